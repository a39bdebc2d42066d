#!/bin/bash
# A/B the working-tree K5 against a saved base library on a GPU box: identical
# trees (tools/k5_ab.py), per-level device times and the 500-tree fit, both
# libraries.  usage: tools/k5_ab_gpu.sh ab/libgk_base.so [out_dir]
set -u
BASE=$1; O=${2:-gpurun_out/ab}; mkdir -p $O
LIB=paper_2305_01886_b200/libgk.so
cp $LIB /tmp/new.so
cp $BASE $LIB
timeout 600 python tools/k5_ab.py save /tmp/a.npz > $O/save.txt 2>&1
timeout 300 python tools/k5_levels.py 1000000 32 > $O/levels_base.txt 2>&1
timeout 300 python tools/rf_fit_bench.py --trees 500 > $O/fit_base.txt 2>&1
cp /tmp/new.so $LIB
timeout 600 python tools/k5_ab.py check /tmp/a.npz > $O/check.txt 2>&1; echo "check rc=$?" >> $O/check.txt
timeout 300 python tools/k5_levels.py 1000000 32 > $O/levels_new.txt 2>&1
timeout 300 python tools/rf_fit_bench.py --trees 500 > $O/fit_new.txt 2>&1
timeout 300 python tools/rf_fit_bench.py --trees 500 >> $O/fit_new.txt 2>&1
tail -n 3 $O/*.txt
