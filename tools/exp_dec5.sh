out=gpurun_out/dec5; mkdir -p $out
ids=0,1,4,5,9,12,14,15
for g in "" even_groups=1 warps=20 ""; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode $ids; done > $out/dbench.jsonl 2>&1
cat $out/dbench.jsonl
