out=gpurun_out/pdl3; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "independent or concurrent" > $out/pytest.log 2>&1; tail -2 $out/pytest.log
