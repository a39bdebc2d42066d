#!/bin/bash
# torchrun 2-rank gloo bench, repeated, with per-rank tracebacks after 60 s (debugging aid)
for k in 1 2 3 4; do
  P=$((29600 + k))
  GK_BENCH_WATCHDOG=60 OMP_NUM_THREADS=2 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
    --master-addr=127.0.0.1 --master-port=$P --local-addr=127.0.0.1 bench.py --gpus 2 --backend gloo \
    --kernels 1000 --cycle-kernels 1000 --steps 2 --warmup 3 --trees 24 --depth 8 --no-rf --no-c4 \
    --cpu-seconds 1 --e2e-steps 1 > gpurun_out/trr$k.out 2> gpurun_out/trr$k.err
  echo "run $k rc=$? lines=$(grep -c '^{' gpurun_out/trr$k.out)"
done
