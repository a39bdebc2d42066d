#!/bin/bash
# One profiling pass on a GPU box (run under gpurun): launch lists and ncu
# --set full captures of the top kernels, into gpurun_out/prof/.  Never reports
# bench values (numbers printed under ncu are not bench numbers).
# usage: tools/profile_round.sh [sweep|c4|k5|all]
set -u
OUT=gpurun_out/prof; mkdir -p $OUT
WHAT=${1:-all}
# config #5 at 100k kernels (76.8M points): same kernels and launch shape as the
# 1M-kernel bench, 1/10 of the points (per-point figures scale)
ARGS="--kernels 100000 --steps 2 --warmup 3 --no-cpu --no-rf --no-c4 --e2e-steps 1 --cycle-kernels 500"
if [[ $WHAT == sweep || $WHAT == all ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_c5.csv python bench.py $ARGS > $OUT/launches.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k23_schedule -s 3 -c 1 \
      -o $OUT/k23_fused_c5 python bench.py $ARGS > $OUT/ncu_k23_fused.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_static -s 3 -c 1 \
      -o $OUT/k1_static_c5 python bench.py $ARGS > $OUT/ncu_k1.log 2>&1
fi
if [[ $WHAT == c4 || $WHAT == all ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_rf_predict -s 1 -c 1 \
      -o $OUT/k4_c4 python bench.py --workload c4 --rows 10000000 --steps 1 --warmup 1 --no-cpu \
      --no-e2e > $OUT/ncu_k4_c4.log 2>&1
fi
if [[ $WHAT == k5 || $WHAT == all ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k5_split_(small|medium)|k5_hist_big|k5_partition" -s 30 -c 8 \
      -o $OUT/k5 python tools/k5_levels.py 1000000 8 > $OUT/ncu_k5.log 2>&1
fi
ls -la $OUT
