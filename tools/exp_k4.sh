out=gpurun_out/k4; mkdir -p $out
for g in "" dyn=2 dyn=1 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py 0 4 8; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
