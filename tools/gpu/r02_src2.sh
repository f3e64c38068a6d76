O=gpurun_out; T=${1:-r02f}
export FZ_COUNT_RUN_COST=64 FZ_COUNT_OUTER_COST=1024
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k5_pairs' -s 1 -c 1 -o $O/${T}_c4 python tools/prof_one.py C4 2 > $O/${T}_ncu.log 2>&1
ncu -i $O/${T}_c4.ncu-rep --page source --csv --print-source sass > $O/${T}_c4_source.csv 2>/dev/null
ncu -i $O/${T}_c4.ncu-rep --page raw --csv > $O/${T}_c4_raw.csv 2>/dev/null
gzip -f $O/${T}_c4_source.csv; rm -f $O/${T}_c4.ncu-rep
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
