out=gpurun_out/clk; mkdir -p $out
for iv in 0.005 0.05 0.005 0.05; do PMRC_CLOCK_INTERVAL=$iv timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$iv', d['ms_per_step'], d['roofline']['kernel_ms'], d['clocks'])"; done > $out/clk.txt 2>&1
timeout 300 python tools/kbench.py >> $out/clk.txt 2>&1
cat $out/clk.txt
