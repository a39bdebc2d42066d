#!/bin/bash
# fused sweep on config #5 (100k kernels) with / without the persisting-L2 window
# (GK_SLAB_L2 lived in gk_sched.cu for this measurement only: the window
# doubled the DRAM writes and cost 4 %, profiles/r2/fused_table_traffic_l2_persist.txt)
# over the reservation-table slabs (GK_SLAB_L2): points/s and one launch's DRAM bytes
for v in 1 0; do
  GK_SLAB_L2=$v timeout 600 python bench.py --kernels 100000 --steps 3 --warmup 3 --no-cpu --no-rf --no-c4 --no-c1 --e2e-steps 1 --cycle-kernels 500 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('GK_SLAB_L2=$v', round(d['value']/1e6,1), 'M pts/s', {k: round(x,1) for k,x in d['kernel_ms'].items()})"
  GK_SLAB_L2=$v timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k23_schedule -s 3 -c 1 \
    python bench.py --kernels 100000 --steps 1 --warmup 3 --no-cpu --no-rf --no-c4 --no-c1 --e2e-steps 1 --cycle-kernels 500 2>/dev/null | grep -E "dram__|gpu__time|lts__"
done
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('persisting L2 max', getattr(p,'persisting_l2_cache_max_size',None), 'L2', p.L2_cache_size)"
