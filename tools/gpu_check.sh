#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (default and the driver's 20-step form), the reference
# arm, the bench's launch list, and an ncu --set full of the encode kernel reduced on the box to
# profiles-ready JSON (tools/ncu_summary.py + tools/ncu_digest.py; the .ncu-rep does not travel).
#   gpurun --timeout 3000 -- 'bash tools/gpu_check.sh <tag> [what...]'
# what: tests smoke bench bench20 ref launches ncu sweep (default: all but sweep)
tag=${1:-r02}; shift
what=${*:-tests smoke bench bench20 ref launches ncu}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $out/nvsmi.txt 2>&1
for w in $what; do
  case $w in
    tests)  timeout 2400 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -3 $out/pytest_gpu.log ;;
    smoke)  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)  timeout 600 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench rc=$?"; cut -c1-400 $out/bench.json ;;
    bench20) timeout 600 python bench.py --steps 20 --warmup 5 > $out/bench20.json 2> $out/bench20.err; echo "bench20 rc=$?"; cut -c1-300 $out/bench20.json ;;
    ref)    timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2> $out/bench_ref.err; echo "ref rc=$?" ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $out/launches.csv python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $out/ncu_launch.log 2>&1
      echo "launches rc=$?"
      python tools/ncu_summary.py launches $out/launches.csv $out/launches_summary.json > /dev/null 2>&1 ;;
    ncu)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmrc_kernel -s 4 -c 1 \
        -o /tmp/encode_full python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $out/ncu_full.log 2>&1
      echo "ncu rc=$?"
      python tools/ncu_summary.py full /tmp/encode_full.ncu-rep $out/ncu_encode_full.json 2231369728 > /dev/null 2>&1
      python tools/ncu_digest.py /tmp/encode_full.ncu-rep $out/ncu_encode_digest.json --rm ;;
    sweep)  timeout 3000 python tools/sweep.py --configs 3,4,5,next1,next2 > $out/sweep.jsonl 2> $out/sweep.err; echo "sweep rc=$?" ;;
  esac
done
