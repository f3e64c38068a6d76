O=gpurun_out
T=r02tail
FZ_LIB_PATH=ab/libfz_tail.so timeout 900 python -m pytest tests -m gpu -q -x -k "count or c4 or staged" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
bash tools/gpu/ab.sh $T "C4 C4t2" ab/libfz_cur.so ab/libfz_tail.so
