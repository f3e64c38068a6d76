O=gpurun_out
T=r02cs5
C="T1 T84b T95 T63 T64 T74"
for pass in 1 2; do
  for L in cs2 cs4 cs5; do FZ_LIB_PATH=ab/libfz_$L.so timeout 300 python tools/ab_time.py $L $C >> $O/${T}_ab.log 2>&1; done
  for spw in 2 3 6 8; do FZ_SLICES_PER_WARP=$spw FZ_LIB_PATH=ab/libfz_cs5.so timeout 300 python tools/ab_time.py cs5_s$spw $C >> $O/${T}_ab.log 2>&1; done
done
