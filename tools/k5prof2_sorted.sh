#!/bin/bash
# the two k5_split_sorted<N> instantiations share ncu's base name: level 15's
# <16> and <32> launches are the 9th and 10th of the batch
set -u
O=${1:-gpurun_out/k5b}; mkdir -p $O
for x in "sorted16_l15 8" "sorted32_l15 9"; do set -- $x
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k5_split_sorted -s $2 -c 1 -o $O/$1 python tools/k5_ncu.py > $O/$1.log 2>&1
done
ls $O
