O=gpurun_out; T=${1:-r02l}
timeout 1500 python bench.py --study f4 > $O/${T}_f4_study.jsonl 2> $O/${T}_f4_study.err
timeout 200 python tools/quick_time.py C3t3 > $O/${T}_c3.log 2>&1
timeout 300 ncu --clock-control none -k regex:'k5_walk' -s 1 -c 1 --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv python tools/prof_one.py C3t3 2 > $O/${T}_c3_ncu.csv 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
