# COUNT pair walk iteration: parity subset, timings, shard balance, shared-memory counters
O=gpurun_out; T=${1:-r02b}
timeout 600 python -m pytest tests -m gpu -x -q -k "count or device_plan or random_small or mid_sharded or edges" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 120 python tools/quick_time.py C4 C4t2 C2c > $O/${T}_quick_time.log 2>&1
timeout 200 python tools/shard_balance.py C4 > $O/${T}_shard_balance.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_pairs' -s 1 -c 1 \
  --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,smsp__inst_executed_op_shared_ld.sum \
  --csv python tools/prof_one.py C4 2 > $O/${T}_c4_smem.csv 2>&1
