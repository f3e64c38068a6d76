O=gpurun_out
T=r02ab2
bash tools/gpu/ab.sh $T "C4" ab/libfz_desc1024.so ab/libfz_addr.so
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_runs' -s 1 -c 1 -o $O/${T}_c4 env FZ_LIB_PATH=ab/libfz_addr.so python tools/prof_one.py C4 2 > /dev/null 2>&1
ncu -i $O/${T}_c4.ncu-rep --page raw --csv > $O/${T}_c4_raw.csv 2>/dev/null
ncu -i $O/${T}_c4.ncu-rep --page source --csv --print-source sass > $O/${T}_c4_source.csv 2>/dev/null
gzip -f $O/${T}_c4_source.csv; rm -f $O/${T}_c4.ncu-rep
FZ_LIB_PATH=ab/libfz_ws.so timeout 900 python -m pytest tests -m gpu -q -x -k "materialize or table1 or random or mid or word or c2" > $O/${T}_tests_ws.log 2>&1; echo "rc=$?" >> $O/${T}_tests_ws.log
bash tools/gpu/ab.sh ${T}m "T95 T94 T1 T63 C2" ab/libfz_addr.so ab/libfz_ws.so
FZ_WORD_STREAM=1 bash tools/gpu/ab.sh ${T}w "T1 C2 T63" ab/libfz_ws.so
