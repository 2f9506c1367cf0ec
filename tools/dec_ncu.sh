#!/bin/bash
# Decode (config 4) timing variants + one ncu --set full capture of the decode kernel.
out=gpurun_out/${1:-dec}; mkdir -p $out
ids=0,1,4,5,9,12,14,15
timeout 300 python tools/dbench.py decode $ids > $out/dbench.jsonl 2>&1
for g in ${VARIANTS}; do
  PMRC_GEN=$g timeout 600 python tools/dbench.py decode $ids >> $out/dbench.jsonl 2>&1
done
cat $out/dbench.jsonl
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pmrc_kernel -s 3 -c 1 \
  -o $out/decode_full python tools/dbench.py decode $ids > $out/ncu_full.log 2>&1
echo "ncu rc=$?"
fi
