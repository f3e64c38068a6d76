O=gpurun_out; T=${1:-r02q}
timeout 300 python -m pytest tests -m gpu -x -q -k "count" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/count_tune.py b96:g3072:t128 > $O/${T}_tune.log 2>&1
timeout 300 python tools/count_tune.py --t2 b96:g3072:t128 > $O/${T}_tune_t2.log 2>&1
(cd ab/r1 && timeout 300 python tools/quick_time.py C4 C4t2 C3t2 C2h > ../../$O/${T}_r1.log 2>&1)
timeout 300 python tools/quick_time.py C4 C4t2 C3t2 C2h > $O/${T}_head.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_walk' -s 1 -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --csv python tools/prof_one.py C3t2 2 > $O/${T}_c3t2_head.csv 2>&1
(cd ab/r1 && timeout 300 ncu --clock-control none -k regex:'k5_walk' -s 1 -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --csv python ../../tools/prof_one.py C3t2 2 > ../../$O/${T}_c3t2_r1.csv 2>&1)
