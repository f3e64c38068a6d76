O=gpurun_out
T=r02cs
FZ_LIB_PATH=ab/libfz_cs.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
C="T95 T94 T1 T63 T74 C2 C3t2 C3t3"
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/ab_time.py addr $C >> $O/${T}_ab.log 2>&1
for spw in 16 8 4; do
  for b in 1 4 16; do
    FZ_ROW_BETA=$b FZ_SLICES_PER_WARP=$spw FZ_LIB_PATH=ab/libfz_cs.so timeout 300 python tools/ab_time.py cs_b${b}_s${spw} $C >> $O/${T}_ab.log 2>&1
  done
done
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/ab_time.py addr $C >> $O/${T}_ab.log 2>&1
