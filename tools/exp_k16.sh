out=gpurun_out/k16; mkdir -p $out
for g in "" layout=1,dyn=2 layout=1,dyn=1; do PMRC_GEN=$g timeout 300 python tools/kbench.py 0 16 32; done > $out/kbench.jsonl 2>&1
for g in "" layout=1,dyn=2; do PMRC_GEN=$g timeout 300 python tools/kbench.py 2 8 16 262144; done >> $out/kbench.jsonl 2>&1
PMRC_GEN=dyn=2 timeout 300 python tools/dbench.py decode 0,1,4,5,9,12,14,15 >> $out/kbench.jsonl 2>&1
timeout 300 python tools/dbench.py decode 0,1,4,5,9,12,14,15 >> $out/kbench.jsonl 2>&1
cat $out/kbench.jsonl
