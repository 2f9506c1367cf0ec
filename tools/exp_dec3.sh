out=gpurun_out/dec3; mkdir -p $out
ids=0,1,4,5,9,12,14,15
for g in trace=1 trace=1,cta_sync=1,warps=20; do PMRC_GEN=$g timeout 300 python tools/dec_trace.py; done > $out/trace.txt 2>&1
for g in "" team=7,warps=14 team=7,warps=21 team=7,warps=21,cta_sync=1 team=7,warps=14,max_rows=16 team=7,warps=21,max_rows=16 team=7,warps=21,max_rows=16,cta_sync=1 team=7,warps=28,max_rows=16; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode $ids; done > $out/dbench.jsonl 2>&1
cat $out/trace.txt $out/dbench.jsonl
