out=gpurun_out/dyn1; mkdir -p $out
for g in "" dyn1=1 "" dyn1=1; do
 PMRC_GEN=$g timeout 300 python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14
 PMRC_GEN=$g timeout 300 python tools/dbench.py repair 6 0,1,2,3,4,5,7,8,9,10,11,13,14,15
 PMRC_GEN=$g timeout 300 python tools/kbench.py 3 8 16
done > $out/r.jsonl 2>&1
cat $out/r.jsonl
