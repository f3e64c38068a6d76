O=gpurun_out
T=r02w3
bash tools/gpu/ab.sh $T "T1 T84b T94 T95 T74" ab/libfz_cur.so ab/libfz_w3.so
FZ_LIB_PATH=ab/libfz_cur.so timeout 300 python tools/table1_bench.py --csv > $O/${T}_t1_cur.csv 2>&1
FZ_LIB_PATH=ab/libfz_w3.so timeout 300 python tools/table1_bench.py --csv > $O/${T}_t1_w3.csv 2>&1
