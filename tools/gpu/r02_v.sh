O=gpurun_out; T=${1:-r02v}
timeout 600 python -m pytest tests -m gpu -x -q -k "count or device_plan" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/count_tune.py b96:g3072:t128 b64:g1024:t128 > $O/${T}_tune.log 2>&1
timeout 300 python tools/count_tune.py --t2 b96:g3072:t128 > $O/${T}_tune_t2.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_runs' -s 1 -c 1 --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg --csv python tools/prof_one.py C4 2 > $O/${T}_c4.csv 2>&1
