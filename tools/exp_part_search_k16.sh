# partition search on the k = 16 encodes (multi-stage groups): A/B at config 5's size
out=gpurun_out/part16; mkdir -p $out
for rep in 1 2; do
  for kind in 0 2; do
    for g in "enc_part_search=0" "part_search=-200"; do
      PMRC_GEN="$g" timeout 900 python tools/kbench.py $kind 16 32 1048576 8589934592 >> $out/enc_k16.jsonl 2>>$out/err.log
    done
  done
done
cat $out/enc_k16.jsonl; tail -3 $out/err.log
