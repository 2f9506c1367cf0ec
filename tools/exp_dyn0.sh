out=gpurun_out/dyn0; mkdir -p $out
for g in "" dyn=1 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py 0 16 32; done > $out/kbench.jsonl 2>&1
for g in "" dyn=1; do PMRC_GEN=$g timeout 300 python tools/kbench.py 2 16 32; done >> $out/kbench.jsonl 2>&1
for g in layout=0 layout=0,dyn=1; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done >> $out/kbench.jsonl 2>&1
cat $out/kbench.jsonl
