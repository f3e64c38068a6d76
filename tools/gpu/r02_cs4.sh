O=gpurun_out
T=r02cs4
FZ_LIB_PATH=ab/libfz_cs4.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
C="T95 T94 T1 T63 T74 C2 C2h C3t2 C3t3 C4"
for pass in 1 2; do
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/ab_time.py addr $C >> $O/${T}_ab.log 2>&1
FZ_LIB_PATH=ab/libfz_cs4.so timeout 300 python tools/ab_time.py cs4 $C >> $O/${T}_ab.log 2>&1
done
FZ_LIB_PATH=ab/libfz_cs4.so timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/table1_bench.py > $O/${T}_table1_addr.log 2>&1
