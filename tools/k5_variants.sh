#!/bin/bash
# K5 build variants on a GPU box: per GK_NVCC_EXTRA variant, rebuild, per-level
# device times of one 32-tree batch and the 500-tree fit; the default build is
# restored at the end.  usage: tools/k5_variants.sh OUT "variant1" "variant2" ...
set -u
O=$1; shift; mkdir -p $O
for v in "$@"; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9_=\n' '_')
  GK_NVCC_EXTRA="$v" python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null || { echo "build failed: $v"; continue; }
  echo "=== variant '$v'" > $O/var_$tag.txt
  timeout 300 python tools/k5_levels.py 1000000 32 | tail -1 >> $O/var_$tag.txt 2>&1
  timeout 300 python tools/rf_fit_bench.py --trees 500 >> $O/var_$tag.txt 2>&1
done
python -c "from paper_2305_01886_b200 import build as B; B.build(force=True)" > /dev/null
cat $O/var_*.txt
