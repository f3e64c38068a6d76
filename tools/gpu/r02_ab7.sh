O=gpurun_out
T=r02ab7
bash tools/gpu/ab.sh ${T} "T95 T94 T1 T63 T74 C2 C3t2" ab/libfz_addr.so ab/libfz_n.so ab/libfz_u.so ab/libfz_p.so
for spw in 24 32; do
  for lib in ab/libfz_n.so ab/libfz_u.so ab/libfz_p.so; do
    FZ_SLICES_PER_WARP=$spw FZ_LIB_PATH=$lib timeout 300 python tools/ab_time.py $(basename $lib .so)_spw$spw T95 T1 T63 C2 >> $O/${T}_spw.log 2>&1
  done
done
