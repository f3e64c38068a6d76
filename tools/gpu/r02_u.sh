O=gpurun_out; T=${1:-r02u}
ncap() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 1 -c 1 -o $O/${T}_$1 python tools/prof_one.py $3 2 > /dev/null 2>&1; ncu -i $O/${T}_$1.ncu-rep --page source --csv --print-source sass > $O/${T}_$1_source.csv 2>/dev/null; ncu -i $O/${T}_$1.ncu-rep --page raw --csv > $O/${T}_$1_raw.csv 2>/dev/null; gzip -f $O/${T}_$1_source.csv; rm -f $O/${T}_$1.ncu-rep; }
ncap c4 k5_runs C4
ncap t95 k5_walk T95
ncap c3t3 k5_walk C3t3
timeout 1500 python tools/parity_stress.py 20000 20000 900 > $O/${T}_stress.log 2>&1
