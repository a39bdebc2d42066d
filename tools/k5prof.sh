#!/bin/bash
# K5 profiling pass (run under gpurun): launch list of one 32-tree batch and
# ncu --set full captures of the deep-level split kernels.
set -u
O=${1:-gpurun_out/k5p}; mkdir -p $O
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches.csv python tools/k5_ncu.py > $O/l.log 2>&1
cap() {  # name kernel skip
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$2 -s $3 -c 1 -o $O/$1 python tools/k5_ncu.py > $O/$1.log 2>&1
}
cap sorted_l15 k5_split_sorted 4
cap rank_l14 k5_split_rank 3
cap mid_l12 k5_split_mid 7
cap med_l9 k5_split_medium 4
cap big_l3 k5_hist_big 3
cap part_l5 k5_partition 5
ls $O
