out=gpurun_out/pdl2; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "independent or concurrent" > $out/pytest.log 2>&1; tail -2 $out/pytest.log
timeout 900 python tools/sweep.py --configs 4 > $out/sweep4.jsonl 2> $out/sweep4.err
for g in "" pdl=2 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/kbench.jsonl 2>&1
grep per-stripe $out/sweep4.jsonl | cut -c1-600; cat $out/kbench.jsonl
