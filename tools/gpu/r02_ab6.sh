O=gpurun_out
T=r02ab6
L=ab/libfz_addr.so
for pass in 1 2; do
  for spw in 16 24 32 64 128; do
    FZ_SLICES_PER_WARP=$spw FZ_LIB_PATH=$L timeout 300 python tools/ab_time.py spw$spw T95 T94 T1 T63 T74 C2 C3t2 >> $O/${T}_ab.log 2>&1
  done
done
