#!/bin/bash
# One profiling pass on a GPU box (run under gpurun): launch list, ncu --set full
# of the top kernels, clocks, into gpurun_out/prof/.  Never reports bench values.
set -u
OUT=gpurun_out/prof; mkdir -p $OUT
ARGS="--steps 2 --warmup 3 --no-cpu --no-rf"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/launches.log 2>&1
for k in k23_schedule k4_rf_predict k1_static; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $OUT/$k python bench.py $ARGS > $OUT/ncu_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k5_ -c 12 \
    -o $OUT/k5 python tools/rf_fit_bench.py --rows 1000000 --trees 8 > $OUT/ncu_k5.log 2>&1
ls -la $OUT
