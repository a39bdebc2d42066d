#!/bin/bash
# K5 build-knob sweep (run on the GPU box): per variant rebuild libgk.so with
# the given -D flags, then the per-level device times of one 32-tree batch
# (tools/k5_levels.py) and the 500-tree fit wall time.
# Usage: tools/sweep_k5.sh "" "-DGK_MED_MINB=4" ...
mkdir -p gpurun_out
for v in "$@"; do
  echo "=== variant: '$v'"
  GK_NVCC_EXTRA="$v" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null || exit 1
  timeout 300 python tools/k5_levels.py 1000000 32 2>/dev/null | tail -1
  timeout 300 python tools/rf_fit_bench.py --trees 500
  timeout 300 python tools/rf_fit_bench.py --trees 500
done
python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
