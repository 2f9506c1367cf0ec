out=gpurun_out/decr; mkdir -p $out
for g in "" cse_restarts=4 ""; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode 0,1,4,5,9,12,14,15; PMRC_GEN=$g timeout 300 python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14; done > $out/d.jsonl 2>&1
cat $out/d.jsonl
