O=gpurun_out
T=r02ws3
FZ_LIB_PATH=ab/libfz_ws3.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
bash tools/gpu/ab.sh $T "T95 T94 T63 T74 T1 C2 C2h C3t3 C3t2" ab/libfz_cur.so ab/libfz_ws3.so
