# MBR k=8 parity-node repairs: how much does the helper set change the kernel time, and which shape fixes the slow ones
out=gpurun_out/mbrrep; mkdir -p $out
H1=0,1,3,4,5,6,7,8,9,10,11,12,13,15
H2=0,1,2,3,4,5,6,7,8,9,11,12,13,15
for g in "" "warps=12,team=2,max_rows=16" "team=2,max_rows=16,warps=8,nbuf=2" "team=2,max_rows=16,warps=12,net_in=8" "team=2,max_rows=16,warps=10,nbuf=3"; do
  for H in $H1 $H2; do
    KIND=2 S=262144 PMRC_GEN="$g" timeout 300 python tools/dbench.py repair 14 $H >> $out/rep14.jsonl 2>>$out/err.log
  done
done
# other lost nodes / helper sets in the default shape
for spec in "14 0,1,2,3,4,5,6,7,8,9,10,11,12,13" "9 0,1,2,3,4,5,6,7,8,10,11,12,13,14" "9 0,1,2,3,4,5,7,8,10,11,12,13,14,15" "15 0,2,3,4,5,6,7,8,9,10,11,12,13,14" "12 1,2,3,4,5,6,7,8,9,10,11,13,14,15" "8 0,1,2,3,4,5,6,7,9,10,11,12,13,14"; do
  set -- $spec
  KIND=2 S=262144 timeout 300 python tools/dbench.py repair $1 $2 >> $out/others.jsonl 2>>$out/err.log
done
cat $out/rep14.jsonl $out/others.jsonl
