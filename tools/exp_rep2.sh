out=gpurun_out/rep2; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 300 python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14
timeout 300 python tools/dbench.py repair 8 0,1,2,3,4,5,6,9,10,11,12,13,14,15
