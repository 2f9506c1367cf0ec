out=gpurun_out/w16w; mkdir -p $out
for g in "" warps=16,smem_kib=226 warps=14,smem_kib=226 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
