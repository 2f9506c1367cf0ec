out=gpurun_out/mbrd; mkdir -p $out
for g in "" dyn=0,nbuf=3 warps=24 in_block=24 dyn=0 warps=8 ""; do PMRC_GEN=$g KIND=2 S=262144 timeout 300 python tools/dbench.py decode 0,1,4,5,6,7,11,14; done > $out/d.jsonl 2>&1
cat $out/d.jsonl
