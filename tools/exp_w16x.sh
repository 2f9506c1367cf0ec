out=gpurun_out/w16x; mkdir -p $out
G=warps=16,smem_kib=226
for g in "" $G; do
 for a in "2 8 16 262144" "3 8 16" "0 4 8" "1 8 16" "2 4 8"; do PMRC_GEN=$g timeout 300 python tools/kbench.py $a; done
 PMRC_GEN=$g timeout 300 python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14
 PMRC_GEN=$g timeout 300 python tools/dbench.py repair 6 0,1,2,3,4,5,7,8,9,10,11,13,14,15
 PMRC_GEN=$g timeout 300 python tools/w16bench.py
done > $out/k.jsonl 2>&1
cat $out/k.jsonl
