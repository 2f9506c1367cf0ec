#!/bin/bash
# generator-variant experiment: parity tests + kernel timing of PMRC_GEN variants + DRAM bytes
#   bash tools/exp_layout.sh <tag> "<variant> <variant> ..." "<ncu variants>"
out=gpurun_out/$1; mkdir -p $out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest.log
fi
for g in $2; do
  PMRC_GEN=$g timeout 300 python tools/kbench.py >> $out/kbench.jsonl 2>>$out/kbench.err
done
cat $out/kbench.jsonl
for g in $3; do
  PMRC_GEN=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active --clock-control none -k regex:pmrc_kernel -s 3 -c 1 python tools/kbench.py > $out/ncu_$g.log 2>&1
  echo "== $g"; grep -E "dram__|gpu__time|lts__|pipe_alu" $out/ncu_$g.log
done
