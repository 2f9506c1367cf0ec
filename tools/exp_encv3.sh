out=gpurun_out/encv3; mkdir -p $out
for g in "" fence=0 tr_unroll=2 l2_shared=2 l2_shared=-1 team=1 max_rows=4 ""; do PMRC_GEN=$g timeout 300 python tools/kbench.py; done > $out/k.jsonl 2>&1
cat $out/k.jsonl
