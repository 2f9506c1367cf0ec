#!/bin/bash
# Build-and-measure variants of the runtime kernel on the GPU box (the box's copy of the repo is
# scratch, so rlc.cu is edited in place there): each argument is "name|sed-expression".
#   gpurun -- 'bash tools/rt_variants.sh <tag> "base|" "d6|s/constexpr int D = 4;/constexpr int D = 6;/"'
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
src=paper_1412_3022_b200/csrc/rt/rlc.cu
cp $src /tmp/rlc_orig.cu
for v in "$@"; do
  name=${v%%|*}; expr=${v#*|}
  cp /tmp/rlc_orig.cu $src
  [ -n "$expr" ] && sed -i -e "$expr" $src
  python -c "import paper_1412_3022_b200.build as b; b.build_lib(force=True)" > $out/build_$name.log 2>&1 || { echo "$name build failed"; continue; }
  timeout 600 python tools/rtbench.py ${RTB_WHAT:-all} 2>/dev/null | sed "s/^{/{\"variant\": \"$name\", /" >> $out/variants.jsonl
  echo "$name done"
done
cp /tmp/rlc_orig.cu $src
