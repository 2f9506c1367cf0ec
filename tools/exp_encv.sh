out=gpurun_out/encv; mkdir -p $out
for g in "" net_in=14 cse_restarts=4 own_first=1 net_in=5 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
