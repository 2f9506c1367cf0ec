out=gpurun_out/dec2; mkdir -p $out
ids=0,1,4,5,9,12,14,15
for g in "" cta_sync=1 warps=20 "cta_sync=1,warps=20"; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode $ids; done > $out/dbench.jsonl 2>&1
for g in "" cta_sync=1; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/kbench.jsonl 2>&1
cat $out/*.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "decode or repair" > $out/pytest.log 2>&1; tail -3 $out/pytest.log
