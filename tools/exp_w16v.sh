out=gpurun_out/w16v; mkdir -p $out
for g in "" max_rows=8 in_block=12 in_block=6 cse_restarts=4; do PMRC_GEN=$g timeout 300 python tools/w16bench.py; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
