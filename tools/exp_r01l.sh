out=gpurun_out/r01l; mkdir -p $out
bash tools/gpu_check.sh r01l tests smoke bench launches ncu
timeout 1500 python tools/sweep.py --configs 3,4,5,next1 --sizes 64,1024 > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
