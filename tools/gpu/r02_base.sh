# round-2 baseline at the round-1 HEAD: quick timings, shard balance, C4 COUNT shared-memory counters
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r02a_smi.txt 2>&1
timeout 300 python tools/quick_time.py C2 C3t3 C4 C4t2 T1 > $O/r02a_quick_time.log 2>&1
timeout 300 python tools/shard_balance.py > $O/r02a_shard_balance.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_walk' -s 1 -c 1 \
  --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum \
  --csv python tools/prof_one.py C4 2 > $O/r02a_c4_smem.csv 2>&1
