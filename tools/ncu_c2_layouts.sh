#!/bin/bash
# ncu counters of the config #2 fused sweep for each walk layout (A/B evidence).
M=l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed
mkdir -p gpurun_out/ncu_layouts
i=0
for v in ${VARIANTS:-"GK_FUSED_COMPACT=0" "GK_FUSED_COMPACT=1"}; do
  env $v timeout 600 ncu --metrics $M --clock-control none -k regex:k23_schedule --launch-skip 2 --launch-count 1 --csv \
    --log-file gpurun_out/ncu_layouts/$i.csv python bench.py --no-cpu --no-rf --steps 1 --warmup 3 > /dev/null 2>&1
  echo "$v" > gpurun_out/ncu_layouts/$i.env
  i=$((i+1))
done
