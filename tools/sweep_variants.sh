#!/bin/bash
# Build libgk variants (-D knobs) and time the stages of the c2 workload.
# usage: tools/sweep_variants.sh "<flags1>" "<flags2>" ...
for f in "$@"; do
  GK_NVCC_EXTRA="$f" python -m paper_2305_01886_b200.build --force > /dev/null || { echo "build failed: $f"; continue; }
  for rep in 1 2; do
    echo -n "[$f] "; NK=${NK:-10000} RF=${RF:-1} timeout 200 python tools/time_stages.py 2>&1 | tail -1
  done
done
python -m paper_2305_01886_b200.build --force > /dev/null
