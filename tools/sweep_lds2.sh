#!/bin/bash
# gk_block2 walk with 3 vs 2 shared-memory feature loads per block (GK_B2_LDS2):
# fused sweep and two-kernel walk on config #5 (100k kernels), K4 on config #4
for v in 0 1; do
  GK_NVCC_EXTRA="-DGK_B2_LDS2=$v" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
  for fused in 1 0; do
    GK_SWEEP_FUSED=$fused timeout 600 python bench.py --kernels 100000 --steps 3 --warmup 3 --no-cpu --no-rf --no-c4 --no-c1 --e2e-steps 1 --cycle-kernels 500 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('LDS2=$v fused=$fused', round(d['value']/1e6,1), 'M pts/s', {k: round(v,1) for k,v in d['kernel_ms'].items()})"
  done
  timeout 600 python bench.py --workload c4 --rows 20000000 --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('LDS2=$v c4', round(d['value']/1e6,1), 'M rows/s')"
done
python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
