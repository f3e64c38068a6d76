O=gpurun_out; T=${1:-r02m}
timeout 200 python tools/quick_time.py C3t3 C3t2 C2h > $O/${T}_c3.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_walk' -s 1 -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active --csv python tools/prof_one.py C3t3 2 > $O/${T}_c3_ncu.csv 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
