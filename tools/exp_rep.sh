out=gpurun_out/rep; mkdir -p $out
for g in "" nbuf=3,dyn=0 in_block=24 warps=16 nbuf=3,dyn=0,warps=8 dyn=2 ""; do PMRC_GEN=$g timeout 300 python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14; done > $out/r.jsonl 2>&1
cat $out/r.jsonl
