set -u
O=gpurun_out/k5p; mkdir -p $O
timeout 300 python tools/k5_levels.py 1000000 32 > $O/levels.txt 2>&1
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,launch__grid_size,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_atom.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file $O/launches.csv python tools/k5_ncu.py > $O/l.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k5_split_small -s 4 -c 1 -o $O/small_l15 python tools/k5_ncu.py > $O/s.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k5_split_medium -s 7 -c 1 -o $O/med_l12 python tools/k5_ncu.py > $O/m.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k5_split_medium -s 2 -c 1 -o $O/med_l7 python tools/k5_ncu.py > $O/m7.log 2>&1
ls -la $O
