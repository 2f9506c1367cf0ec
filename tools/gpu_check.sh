#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list, ncu --set full of the encode kernel.
#   gpurun --timeout 1800 -- 'bash tools/gpu_check.sh <tag> [what...]'
# what: tests smoke bench launches ncu sweep (default: all but sweep)
tag=${1:-r01}; shift
what=${*:-tests smoke bench launches ncu}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/nvsmi.txt 2>&1
for w in $what; do
  case $w in
    tests)  timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "tests rc=$?" ;;
    smoke)  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)  timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cat $out/bench.json ;;
    ref)    timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?" ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $out/ncu_launch.log 2>&1
      echo "launches rc=$?" ;;
    ncu)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmrc_kernel -s 4 -c 1 \
        -o $out/encode_full python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $out/ncu_full.log 2>&1
      echo "ncu rc=$?" ;;
    sweep)  timeout 1200 python tools/sweep.py > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?" ;;
  esac
done
tail -3 $out/pytest_gpu.log 2>/dev/null
