out=gpurun_out/fin2; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 300 python tools/w16bench.py > $out/w16.jsonl 2>&1
timeout 600 python tools/sweep.py --configs next1 > $out/next1.jsonl 2>&1
cat $out/w16.jsonl; cut -c1-200 $out/next1.jsonl
