out=gpurun_out/r01n; mkdir -p $out
bash tools/gpu_check.sh r01n tests smoke bench launches ncu ref
timeout 1500 python tools/sweep.py --configs 3,4,5,next1 --sizes 64,1024 > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?"
timeout 300 python tools/w16bench.py > $out/w16.jsonl 2>&1
