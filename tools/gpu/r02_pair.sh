O=gpurun_out
T=r02pair
for L in p0 p1; do FZ_LIB_PATH=ab/libfz_$L.so timeout 900 python -m pytest tests -m gpu -q -x -k "count or c4 or staged" > $O/${T}_tests_$L.log 2>&1; echo "rc=$?" >> $O/${T}_tests_$L.log; done
bash tools/gpu/ab.sh $T "C4 C4t2" paper_2407_20474_b200/libfz.so ab/libfz_p0.so ab/libfz_p1.so
