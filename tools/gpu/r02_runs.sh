O=gpurun_out; T=${1:-r02o}
timeout 600 python -m pytest tests -m gpu -x -q -k "count or device_plan or random_small or mid_sharded or edges" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
FZ_COUNT_WALK=pairs timeout 600 python -m pytest tests -m gpu -x -q -k "count" > $O/${T}_tests_pairs.log 2>&1; echo "rc=$?" >> $O/${T}_tests_pairs.log
(cd ab/r1 && timeout 300 python tools/quick_time.py C4 > ../../$O/${T}_r1.log 2>&1)
timeout 500 python tools/count_tune.py b64:g1024:t128 b32:g512:t128 b16:g256:t128 > $O/${T}_tune_runs.log 2>&1
FZ_COUNT_WALK=pairs timeout 300 python tools/count_tune.py b64:g1024:t128 > $O/${T}_tune_pairs.log 2>&1
timeout 300 python tools/count_tune.py --t2 b64:g1024:t128 b32:g512:t128 > $O/${T}_tune_t2.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_runs' -s 1 -c 1 \
  --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,smsp__inst_executed_op_shared_ld.sum,sm__cycles_active.avg \
  --csv python tools/prof_one.py C4 2 > $O/${T}_c4_smem.csv 2>&1
