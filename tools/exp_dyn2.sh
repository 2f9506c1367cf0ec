out=gpurun_out/dyn2; mkdir -p $out
for g in "" dyn=0; do PMRC_GEN=$g timeout 900 python tools/sweep.py --configs 3,4 ; done > $out/sweep.jsonl 2> $out/sweep.err
cat $out/sweep.jsonl
