#!/bin/bash
# One profiling pass on a GPU box (run under gpurun): launch list, ncu --set full
# of the top kernels, into gpurun_out/prof/.  Never reports bench values.
# usage: tools/profile_round.sh [sweep|k5|c4|all]
set -u
OUT=gpurun_out/prof; mkdir -p $OUT
WHAT=${1:-all}
ARGS="--steps 2 --warmup 3 --no-cpu --no-rf"
if [[ $WHAT == sweep || $WHAT == all ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/launches.log 2>&1
  # fused sweep (the dominant kernel of the default bench), then K1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k23_schedule -s 2 -c 1 \
      -o $OUT/k23_fused python bench.py $ARGS > $OUT/ncu_k23_fused.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_static -s 2 -c 1 \
      -o $OUT/k1_static python bench.py $ARGS > $OUT/ncu_k1.log 2>&1
fi
if [[ $WHAT == c4 || $WHAT == all ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_rf_predict -s 3 -c 1 \
      -o $OUT/k4_c4 python bench.py --workload c4 --rows 2000000 $ARGS > $OUT/ncu_k4_c4.log 2>&1
fi
if [[ $WHAT == k5 || $WHAT == all ]]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k5_ -c 12 \
      -o $OUT/k5 python tools/rf_fit_bench.py --rows 1000000 --trees 8 > $OUT/ncu_k5.log 2>&1
fi
ls -la $OUT
