out=gpurun_out/k16b; mkdir -p $out
for g in "" max_rows=16,team=4,warps=16 max_rows=16,team=4,warps=16,layout=0 max_rows=16,team=4,warps=16,dyn=2; do PMRC_GEN=$g timeout 300 python tools/kbench.py 0 16 32; done > $out/kbench.jsonl 2>&1
cat $out/kbench.jsonl
