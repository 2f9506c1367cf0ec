out=gpurun_out/tpc; mkdir -p $out
PMRC_GEN=trace=1 timeout 300 python tools/tpc_trace.py > $out/enc.txt 2>&1
PMRC_GEN=trace=1,dyn=0 timeout 300 python tools/tpc_trace.py --decode > $out/dec.txt 2>&1
cat $out/enc.txt $out/dec.txt
