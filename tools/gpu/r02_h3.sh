O=gpurun_out
T=r02h3
for pass in 1 2; do
for L in base h43 h33; do FZ_LIB_PATH=ab/libfz_$L.so timeout 300 python tools/ab_time.py $L C3t3 C3t2 C2h C2c >> $O/${T}_ab.log 2>&1; done
done
FZ_LIB_PATH=ab/libfz_h43.so timeout 900 python -m pytest tests -m gpu -q -x -k "hash or c3 or random or table1" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
