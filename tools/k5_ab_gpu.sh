#!/bin/bash
# A/B the working tree's K5 against a base source tree (e.g. `git archive` of a
# commit, built in place) on a GPU box: identical trees (tools/k5_ab.py),
# per-level device times and the 500-tree fit for both.
# usage: tools/k5_ab_gpu.sh BASE_TREE [out_dir]
set -u
BASE=$1; O=${2:-gpurun_out/ab}; mkdir -p $O
(cd $BASE && timeout 600 python tools/k5_ab.py save /tmp/a.npz > /dev/null 2>&1 &&
  timeout 300 python tools/k5_levels.py 1000000 32 > /tmp/levels_base.txt 2>&1 &&
  timeout 300 python tools/rf_fit_bench.py --trees 500 --repeat 3 --streams 4 > /tmp/fit_base.txt 2>&1)
cp /tmp/levels_base.txt /tmp/fit_base.txt $O/
timeout 600 python tools/k5_ab.py check /tmp/a.npz > $O/check.txt 2>&1; echo "check rc=$?" >> $O/check.txt
timeout 300 python tools/k5_levels.py 1000000 32 > $O/levels_new.txt 2>&1
timeout 300 python tools/rf_fit_bench.py --trees 500 --repeat 3 --streams 4 > $O/fit_new.txt 2>&1
cat $O/check.txt
paste <(cut -c1-80 $O/levels_base.txt) <(cut -c40-80 $O/levels_new.txt)
grep -h "^fit" $O/fit_base.txt | sed 's/^/base /'; grep -h "^fit" $O/fit_new.txt | sed 's/^/new  /'
