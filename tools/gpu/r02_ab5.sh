O=gpurun_out
T=r02ab5
L=ab/libfz_addr.so
for pass in 1 2; do
  FZ_LIB_PATH=$L timeout 300 python tools/ab_time.py spw16 T95 T94 T1 T63 T74 C2 C3t2 >> $O/${T}_ab.log 2>&1
  FZ_SLICES_PER_WARP=8 FZ_LIB_PATH=$L timeout 300 python tools/ab_time.py spw8 T95 T94 T1 T63 T74 C2 C3t2 >> $O/${T}_ab.log 2>&1
  FZ_SLICES_PER_WARP=4 FZ_LIB_PATH=$L timeout 300 python tools/ab_time.py spw4 T95 T94 T1 T63 T74 C2 C3t2 >> $O/${T}_ab.log 2>&1
  FZ_ROW_GSS=1 FZ_LIB_PATH=$L timeout 300 python tools/ab_time.py gss T95 T94 T1 T63 T74 C2 C3t2 >> $O/${T}_ab.log 2>&1
done
