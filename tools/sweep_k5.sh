#!/bin/bash
# K5 build-knob sweep (run on the GPU box): per variant rebuild libgk.so with
# the given -D flags, then per-kernel device time (64 trees) and the 128-tree
# fit wall time.  Usage: tools/sweep_k5.sh "-DGK_SMALL_MINB=4 -DGK_MED_MINB=2" "..."
mkdir -p gpurun_out
for v in "$@"; do
  echo "=== $v"
  GK_NVCC_EXTRA="$v" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null || exit 1
  timeout 300 python tools/kernel_profile.py rf 1000000 64 2>/dev/null | grep -E 'wall|k5_split|k5_hist_big'
  timeout 300 python tools/rf_fit_bench.py --trees 128
done
