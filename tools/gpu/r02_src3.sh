O=gpurun_out; T=${1:-r02p}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k5_runs' -s 1 -c 1 -o $O/${T}_c4 python tools/prof_one.py C4 2 > $O/${T}_ncu.log 2>&1
ncu -i $O/${T}_c4.ncu-rep --page source --csv --print-source sass > $O/${T}_c4_source.csv 2>/dev/null
gzip -f $O/${T}_c4_source.csv; rm -f $O/${T}_c4.ncu-rep
timeout 500 python tools/count_tune.py b96:g1024:t128 b128:g2048:t128 b96:g3072:t128 > $O/${T}_tune_runs.log 2>&1
