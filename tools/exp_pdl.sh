out=gpurun_out/pdl; mkdir -p $out
for g in "" pdl=1 pdl=2; do PMRC_GEN=$g timeout 900 python tools/sweep.py --configs 4 2>/dev/null | grep per-stripe | sed "s/^/$g /"; done > $out/sweep.txt 2>&1
cat $out/sweep.txt | cut -c1-400
