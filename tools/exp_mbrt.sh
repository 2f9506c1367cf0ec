out=gpurun_out/mbrt; mkdir -p $out
PMRC_GEN=trace=1 timeout 300 python tools/pace_trace.py 2 8 16 262144 > $out/trace.txt 2>&1
cat $out/trace.txt
