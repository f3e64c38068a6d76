O=gpurun_out
T=r02hf
FZ_LIB_PATH=ab/libfz_hf.so timeout 900 python -m pytest tests -m gpu -q -x -k "hash or c3 or random or table1 or c2 or slice" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
bash tools/gpu/ab.sh $T "C3t3 C3t2 C2h" ab/libfz_cur.so ab/libfz_hf.so
