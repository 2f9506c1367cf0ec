#!/bin/bash
# run tools/sweep.py under several PMRC_GEN variants: bash tools/exp_sweep.sh <tag> <configs> "<variants>" [extra sweep args]
out=gpurun_out/$1; mkdir -p $out
for g in $3; do
  echo "== $g"
  PMRC_GEN=$g timeout 900 python tools/sweep.py --configs $2 $4 2>>$out/err.txt | tee -a $out/sweep.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$g', d['op'], d.get('config',''), d['kind'], d['k'], d['S']>>10, d['ms'], d.get('GBps', d.get('GBps_repaired')), d.get('bit_exact',''))"
done
