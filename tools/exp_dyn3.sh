out=gpurun_out/dyn3; mkdir -p $out
ids=0,1,4,5,9,12,14,15
for g in "" dyn=2; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/kbench.jsonl 2>&1
for g in "" dyn=2; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode $ids; done > $out/dbench.jsonl 2>&1
PMRC_GEN=dyn=2,trace=1 timeout 300 python tools/dec_trace.py > $out/trace.txt 2>&1
cat $out/kbench.jsonl $out/dbench.jsonl $out/trace.txt
PMRC_GEN=dyn=2 timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; tail -3 $out/pytest.log
