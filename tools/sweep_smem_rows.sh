#!/bin/bash
# fused sweep on config #5 (100k kernels) vs GK_SMEM_ROWS (reservation-table rows
# per lane kept in shared memory; 0 = all in the L1-backed global slab): points/s
# and one launch's DRAM bytes (ncu)
for r in "$@"; do
  GK_SMEM_ROWS=$r timeout 600 python bench.py --kernels 100000 --steps 3 --warmup 3 --no-cpu --no-rf --no-c4 --no-c1 --e2e-steps 1 --cycle-kernels 500 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('rows $r', round(d['value']/1e6,1), 'M pts/s', {k: round(x,1) for k,x in d['kernel_ms'].items()})"
  GK_SMEM_ROWS=$r timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k23_schedule -s 3 -c 1 \
    python bench.py --kernels 100000 --steps 1 --warmup 3 --no-cpu --no-rf --no-c4 --no-c1 --e2e-steps 1 --cycle-kernels 500 2>/dev/null | grep -E "dram__|gpu__time"
done
