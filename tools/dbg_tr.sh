#!/bin/bash
# run bench.py as 2 gloo ranks by hand (tracebacks on timeout), debugging aid
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29541 WORLD_SIZE=2 PYTHONFAULTHANDLER=1 OMP_NUM_THREADS=2
ARGS="--gpus 2 --backend gloo --kernels 1000 --cycle-kernels 1000 --steps 2 --warmup 3 --trees 24 --depth 8 --no-rf --no-c4 --cpu-seconds 1 --e2e-steps 1"
for r in 0 1; do
  RANK=$r LOCAL_RANK=$r timeout -s ABRT ${1:-180} python bench.py $ARGS > gpurun_out/tr$r.out 2> gpurun_out/tr$r.err &
done
wait
for r in 0 1; do echo "== rank $r"; grep -v "^\s*File \"/opt\|^Extension" gpurun_out/tr$r.err | tail -25; tail -c 300 gpurun_out/tr$r.out; done
