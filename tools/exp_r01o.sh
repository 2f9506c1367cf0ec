out=gpurun_out/r01o; mkdir -p $out
bash tools/gpu_check.sh r01o tests smoke bench launches ncu
timeout 1500 python tools/sweep.py --configs 3,4,next1 > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
