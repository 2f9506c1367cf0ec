out=gpurun_out/dec6; mkdir -p $out
for g in "" own_first=1 net_in=10 net_in=14 own_first=1,net_in=10 ""; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode 0,1,4,5,9,12,14,15; done > $out/dbench.jsonl 2>&1
cat $out/dbench.jsonl
