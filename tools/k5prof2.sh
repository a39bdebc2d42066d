#!/bin/bash
# K5 binding-unit captures of the current kernel set (run under gpurun): one
# ncu --set full capture per split / partition kernel at the level where it
# carries the most time in one 32-tree batch of config #3 (tools/k5_ncu.py).
set -u
O=${1:-gpurun_out/k5b}; mkdir -p $O
cap() {  # name kernel-regex skip
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$2 -s $3 -c 1 -o $O/$1 python tools/k5_ncu.py > $O/$1.log 2>&1
}
cap sorted16_l15 'k5_split_sorted<16>' 4
cap sorted32_l15 'k5_split_sorted<32>' 4
cap radix_l14 k5_split_radix 3
cap mid_l12 k5_split_mid 7
cap med_l11 k5_split_medium 6
cap big_l3 k5_hist_big 3
cap part_l12 k5_partition 12
ls $O
