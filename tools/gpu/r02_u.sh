O=gpurun_out
T=r02u
for L in u1 u2; do FZ_LIB_PATH=ab/libfz_$L.so timeout 600 python -m pytest tests -m gpu -q -x -k "count or c4 or staged" > $O/${T}_tests_$L.log 2>&1; echo "rc=$?" >> $O/${T}_tests_$L.log; done
bash tools/gpu/ab.sh $T "C4 C4t2 C2c" paper_2407_20474_b200/libfz.so ab/libfz_u1.so ab/libfz_u2.so
