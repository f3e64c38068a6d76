O=gpurun_out
T=r02cs2
FZ_LIB_PATH=ab/libfz_cs2.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
C="T95 T94 T1 T63 T74 C2 C3t2 C3t3"
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/ab_time.py addr $C >> $O/${T}_ab.log 2>&1
FZ_LIB_PATH=ab/libfz_cs2.so timeout 300 python tools/ab_time.py auto $C >> $O/${T}_ab.log 2>&1
for spw in 2 3 4; do
  for b in 16 32 64; do
    FZ_ROW_BETA=$b FZ_SLICES_PER_WARP=$spw FZ_LIB_PATH=ab/libfz_cs2.so timeout 300 python tools/ab_time.py cs_b${b}_s${spw} T95 T94 T1 T63 T74 >> $O/${T}_ab.log 2>&1
  done
done
FZ_LIB_PATH=ab/libfz_cs2.so timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/table1_bench.py > $O/${T}_table1_addr.log 2>&1
