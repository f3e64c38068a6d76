O=gpurun_out
T=r02cs3
for pass in 1 2; do
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/ab_time.py addr C2 C3t2 C3t3 T95 T1 >> $O/${T}_ab.log 2>&1
for L in cs2 cs3; do
  FZ_ROW_BETA=0 FZ_LIB_PATH=ab/libfz_$L.so timeout 300 python tools/ab_time.py ${L}_rows C2 C3t2 C3t3 T95 T1 >> $O/${T}_ab.log 2>&1
  FZ_ROW_BETA=16 FZ_LIB_PATH=ab/libfz_$L.so timeout 300 python tools/ab_time.py ${L}_b16s4 C2 C3t2 C3t3 T95 T1 >> $O/${T}_ab.log 2>&1
  FZ_ROW_BETA=16 FZ_SLICES_PER_WARP=16 FZ_LIB_PATH=ab/libfz_$L.so timeout 300 python tools/ab_time.py ${L}_b16s16 C2 C3t2 C3t3 >> $O/${T}_ab.log 2>&1
  FZ_ROW_BETA=4 FZ_SLICES_PER_WARP=16 FZ_LIB_PATH=ab/libfz_$L.so timeout 300 python tools/ab_time.py ${L}_b4s16 C2 C3t2 C3t3 >> $O/${T}_ab.log 2>&1
done
done
