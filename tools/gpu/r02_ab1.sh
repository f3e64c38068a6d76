O=gpurun_out
T=r02ab1
FZ_LIB_PATH=ab/libfz_desc1024.so timeout 900 python -m pytest tests -m gpu -q -x -k "count or c4 or staged" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
bash tools/gpu/ab.sh $T "C4 C4t2" ab/libfz_head.so ab/libfz_desc1024.so ab/libfz_desc768.so
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/${T}_t95 python tools/prof_one.py T95 2 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/${T}_t1 python tools/prof_one.py T1 2 > /dev/null 2>&1
for r in t95 t1; do
  ncu -i $O/${T}_$r.ncu-rep --page raw --csv > $O/${T}_${r}_raw.csv 2>/dev/null
  ncu -i $O/${T}_$r.ncu-rep --page source --csv --print-source sass > $O/${T}_${r}_source.csv 2>/dev/null
  ncu -i $O/${T}_$r.ncu-rep --page details --csv > $O/${T}_${r}_details.csv 2>/dev/null
  gzip -f $O/${T}_${r}_source.csv
  rm -f $O/${T}_$r.ncu-rep
done
