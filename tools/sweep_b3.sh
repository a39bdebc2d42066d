#!/bin/bash
# K4 on config #4 (20M rows) with the gk_block3 walk at several lock-step widths
# vs the gk_block2 default (run on a GPU box; restores the default build)
for ilp in 2 4 6 8; do
  GK_NVCC_EXTRA="-DGK_RF_B3_ILP=$ilp" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
  GK_WALK_LAYOUT=blocks3 timeout 600 python bench.py --workload c4 --rows 20000000 --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('blocks3 ilp $ilp', round(d['value']/1e6,1), 'M rows/s')"
done
python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
timeout 600 python bench.py --workload c4 --rows 20000000 --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('blocks (default)', round(d['value']/1e6,1), 'M rows/s')"
