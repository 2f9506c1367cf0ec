out=gpurun_out/w16r; mkdir -p $out
for g in "" auto_wide16=0; do PMRC_GEN=$g timeout 300 python tools/kbench.py 0 16 32; PMRC_GEN=$g timeout 300 python tools/kbench.py 2 16 32; done > $out/kbench.jsonl 2>&1
for g in "" dyn=0; do PMRC_GEN=$g timeout 300 python tools/kbench.py 2 4 8; done >> $out/kbench.jsonl 2>&1
cat $out/kbench.jsonl
