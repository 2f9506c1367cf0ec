out=gpurun_out/dec4; mkdir -p $out
for g in trace=1; do PMRC_GEN=$g timeout 300 python tools/dec_trace.py; done > $out/trace.txt 2>&1
cat $out/trace.txt
