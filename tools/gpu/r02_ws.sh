O=gpurun_out; T=${1:-r02h}
timeout 300 python tools/quick_time.py T95 T63 T31 T74 > $O/${T}_ws1.log 2>&1
FZ_WORD_STREAM=0 timeout 300 python tools/quick_time.py T95 T63 T31 T74 > $O/${T}_ws0.log 2>&1
for W in 1 0; do
FZ_WORD_STREAM=$W timeout 300 ncu --clock-control none -k regex:'k5_walk' -s 1 -c 1 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sectors_op_write.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem \
  --csv python tools/prof_one.py T95 2 > $O/${T}_t95_ws$W.csv 2>&1
done
timeout 500 python tools/count_tune.py b64:g1024:t128 > $O/${T}_tune.log 2>&1
timeout 300 python tools/count_tune.py --t2 b64:g1024:t128 > $O/${T}_tune_t2.log 2>&1
