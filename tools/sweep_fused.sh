#!/bin/bash
# fused sweep on config #5 (100k kernels) over build variants (GK_NVCC_EXTRA); restores the default
for v in "$@"; do
  GK_NVCC_EXTRA="$v" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py --kernels 100000 --steps 3 --warmup 3 --no-cpu --no-rf --no-c4 --no-c1 --e2e-steps 1 --cycle-kernels 500 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value']/1e6,1), 'M pts/s', {k: round(x,1) for k,x in d['kernel_ms'].items()})"
done
python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
