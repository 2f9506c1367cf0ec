# partition search of the encode networks (enc_part_search) A/B, and the 12-warp shape for light multi-stage single-group plans
out=gpurun_out/part; mkdir -p $out
for rep in 1 2 3; do
  for g in "enc_part_search=0" "" "enc_part_search=600"; do
    PMRC_GEN="$g" timeout 600 python tools/kbench.py 0 8 16 1048576 1073741824 >> $out/enc_msr8.jsonl 2>>$out/err.log
  done
done
for rep in 1 2; do
  for g in "enc_part_search=0" "" "enc_part_search=600"; do
    PMRC_GEN="$g" timeout 600 python tools/kbench.py 2 8 16 262144 1073741824 >> $out/enc_mbr8.jsonl 2>>$out/err.log
    PMRC_GEN="$g" timeout 600 python tools/kbench.py 0 4 8 1048576 1073741824 >> $out/enc_msr4.jsonl 2>>$out/err.log
  done
done
for spec in "14 0,1,3,4,5,6,7,8,9,10,11,12,13,15" "14 0,1,2,3,4,5,6,7,8,9,11,12,13,15" "9 0,1,2,3,4,5,7,8,10,11,12,13,14,15" "15 0,2,3,4,5,6,7,8,9,10,11,12,13,14" "12 1,2,3,4,5,6,7,8,9,10,11,13,14,15" "8 0,1,2,3,4,5,6,7,9,10,11,12,13,14" "3 0,1,2,4,5,6,7,8,9,10,11,12,13,14" "0 1,2,3,4,5,6,7,8,9,10,11,12,13,15"; do
  set -- $spec
  KIND=2 S=262144 timeout 300 python tools/dbench.py repair $1 $2 >> $out/mbr_repair_12w.jsonl 2>>$out/err.log
done
cat $out/*.jsonl | cut -c1-250; tail -3 $out/err.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "encode or repair or fuzz" 2>&1 | tail -5 > $out/pytest_tail.txt; cat $out/pytest_tail.txt
