#!/bin/bash
# Fused-sweep DRAM write-back vs reservation-table discard mode (run on the GPU
# box): per GK_DISCARD mode, rebuild, then ncu DRAM bytes + duration of one
# fused-sweep launch on the c2 grid (10k kernels) and the bench's kernel_ms.
for d in 0 1 2; do
  echo "=== GK_DISCARD=$d"
  GK_NVCC_EXTRA="-DGK_DISCARD=$d" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null || exit 1
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k23_schedule -s 3 -c 1 python bench.py --workload c2 --steps 2 \
      --warmup 3 --no-cpu --no-rf --e2e-steps 1 2>/dev/null | grep -E "dram__|gpu__time"
  timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu --no-rf --e2e-steps 1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kernel_ms', d['kernel_ms'])"
done
python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
