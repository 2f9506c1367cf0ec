# MBR k=8 parity-node repairs, second pass: shapes for the slow class (helper sets missing a systematic node)
out=gpurun_out/mbrrep2; mkdir -p $out
H1=0,1,3,4,5,6,7,8,9,10,11,12,13,15
H2=0,1,2,3,4,5,6,7,8,9,11,12,13,15
for g in "team=2,max_rows=16,warps=16" "team=2,max_rows=16,warps=14" "team=2,max_rows=16,warps=8,nbuf=3,fence=0" \
    "team=2,max_rows=16,warps=8,nbuf=3,net_in=8" "team=2,max_rows=16,warps=8,nbuf=3,net_in=14" "team=2,max_rows=16,warps=8,nbuf=4" \
    "team=2,max_rows=16,warps=12,nbuf=2,net_in=14" "team=2,max_rows=16,warps=12,tr_unroll=2" "team=2,max_rows=16,warps=8,nbuf=3,dyn=0" "team=2,max_rows=16,warps=12,dyn=0"; do
  for H in $H1 $H2; do
    KIND=2 S=262144 PMRC_GEN="$g" timeout 300 python tools/dbench.py repair 14 $H >> $out/rep14.jsonl 2>>$out/err.log
  done
done
cat $out/rep14.jsonl; tail -3 $out/err.log
