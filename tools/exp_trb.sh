out=gpurun_out/trb; mkdir -p $out
ids=0,1,4,5,9,12,14,15
for g in "" tr_balance=1 "" tr_balance=1; do PMRC_GEN=$g timeout 300 python tools/dbench.py decode $ids; done > $out/dbench.jsonl 2>&1
for g in "" tr_balance=1; do PMRC_GEN=$g timeout 300 python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14; PMRC_GEN=$g timeout 300 python tools/dbench.py repair 6 0,1,2,3,4,5,7,8,9,10,11,13,14,15; done > $out/rbench.jsonl 2>&1
cat $out/*.jsonl
