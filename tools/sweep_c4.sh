#!/bin/bash
# Build libgk variants (-D knobs) and time config #4's K4 on a row subset.
# usage: ROWS=20000000 tools/sweep_c4.sh "<flags1>" "<flags2>" ...
for f in "$@"; do
  GK_NVCC_EXTRA="$f" python -m paper_2305_01886_b200.build --force > /dev/null || { echo "build failed: $f"; continue; }
  echo -n "[$f] "
  timeout 300 python bench.py --workload c4 --rows ${ROWS:-20000000} --no-cpu --no-e2e --steps 3 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M rows/s', round(d['ms_per_step'],1), 'ms')"
done
python -m paper_2305_01886_b200.build --force > /dev/null
