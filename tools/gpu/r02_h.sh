O=gpurun_out
T=r02h2
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
for pass in 1 2; do
FZ_LIB_PATH=ab/libfz_g.so timeout 300 python tools/ab_time.py prev C3t3 C3t2 C2h T95 >> $O/${T}_ab.log 2>&1
timeout 300 python tools/ab_time.py mul3 C3t3 C3t2 C2h T95 >> $O/${T}_ab.log 2>&1
done
