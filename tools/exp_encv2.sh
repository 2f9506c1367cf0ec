out=gpurun_out/encv2; mkdir -p $out
for g in "" cse_restarts=4 cse_restarts=8 cse_restarts=16 "" cse_restarts=4; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
