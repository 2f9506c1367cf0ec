out=gpurun_out/abl; mkdir -p $out
for g in "" debug=1 debug=2 debug=3 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
