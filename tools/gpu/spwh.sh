# HASH slice-queue granularity sweep (FZ_SLICES_PER_WARP)
O=gpurun_out
for k in 8 16 32 64; do FZ_SLICES_PER_WARP=$k timeout 200 python tools/quick_time.py C3t3 C2h C3t4 > $O/spwh_$k.log 2>&1; done
