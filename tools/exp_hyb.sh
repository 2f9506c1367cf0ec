out=gpurun_out/hyb; mkdir -p $out
for g in "" dyn=2,dyn_static=800 dyn=2,dyn_static=900 dyn=2,dyn_static=950 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/kbench.jsonl 2>&1
for g in "" dyn=2,dyn_static=800 dyn=2,dyn_static=900 dyn=2,dyn_static=950; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode 0,1,4,5,9,12,14,15; done >> $out/kbench.jsonl 2>&1
cat $out/kbench.jsonl
PMRC_GEN=dyn=2,dyn_static=900 timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -3 $out/pytest.log
