#!/bin/bash
# Time the config #2 fused sweep under build flags / env knobs.
# usage: tools/sweep_c2.sh "<nvcc flags>|<env assignments>" ...
#   e.g. "-DGK_FUSED_B2_ILP=6|GK_WALK_LAYOUT=blocks GK_FUSED_COMPACT=1"
for spec in "$@"; do
  flags="${spec%%|*}"; envs="${spec#*|}"; [ "$envs" = "$spec" ] && envs=""
  GK_NVCC_EXTRA="$flags" python -m paper_2305_01886_b200.build --force > /dev/null || { echo "build failed: $flags"; continue; }
  for rep in 1 2; do
    echo -n "[$flags | $envs] "
    env $envs timeout 300 python bench.py --no-cpu --no-rf --steps 5 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M pts/s', round(d['kernel_ms']['k23_schedule<fused>'],3), 'ms fused', round(d['cycle_sweep']['ms_per_step'],3), 'ms cycles-only')"
  done
done
python -m paper_2305_01886_b200.build --force > /dev/null
