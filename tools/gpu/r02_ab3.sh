O=gpurun_out
T=r02ab3
FZ_LIB_PATH=ab/libfz_tr.so timeout 900 python -m pytest tests -m gpu -q -x -k "count or c4 or staged" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
bash tools/gpu/ab.sh $T "C4 C4t2" ab/libfz_addr.so ab/libfz_tr.so
bash tools/gpu/ab.sh ${T}m "T95 T94 T1 T63 C2" ab/libfz_addr.so ab/libfz_tr.so
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_runs' -s 1 -c 1 -o $O/${T}_c4 env FZ_LIB_PATH=ab/libfz_tr.so python tools/prof_one.py C4 2 > /dev/null 2>&1
ncu -i $O/${T}_c4.ncu-rep --page raw --csv > $O/${T}_c4_raw.csv 2>/dev/null
ncu -i $O/${T}_c4.ncu-rep --page source --csv --print-source sass > $O/${T}_c4_source.csv 2>/dev/null
gzip -f $O/${T}_c4_source.csv; rm -f $O/${T}_c4.ncu-rep
