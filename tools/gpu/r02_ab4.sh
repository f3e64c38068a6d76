O=gpurun_out
T=r02ab4
FZ_LIB_PATH=ab/libfz_cur1.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
bash tools/gpu/ab.sh ${T}m "T95 T94 T1 T63 T74 C2 C3t2 C4" ab/libfz_addr.so ab/libfz_cur1.so ab/libfz_cur4.so
FZ_LIB_PATH=ab/libfz_cur1.so timeout 300 python tools/table1_bench.py > $O/${T}_table1_cur1.log 2>&1
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/table1_bench.py > $O/${T}_table1_addr.log 2>&1
