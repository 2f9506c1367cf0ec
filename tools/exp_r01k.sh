out=gpurun_out/r01k; mkdir -p $out
bash tools/gpu_check.sh r01k tests bench
timeout 900 python tools/sweep.py --configs 3,4 > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
ids=0,1,4,5,9,12,14,15
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmrc_kernel -s 3 -c 1 \
  -o $out/decode_full python tools/dbench.py decode $ids > $out/ncu_dec.log 2>&1
echo "ncu rc=$?"
