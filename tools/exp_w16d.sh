out=gpurun_out/w16d; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "concurrent_streams" > $out/pytest.log 2>&1; tail -2 $out/pytest.log
for g in "" dyn=2 ""; do PMRC_GEN=$g timeout 300 python tools/w16bench.py; done > $out/w16.jsonl 2>&1
cat $out/w16.jsonl
