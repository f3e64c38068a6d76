# COUNT slice-queue granularity sweep on C4 (FZ_SLICES_PER_WARP)
O=gpurun_out
for k in 32 64 128; do FZ_SLICES_PER_WARP=$k timeout 200 python bench.py --config C4 --steps 10 --no-cpu --no-e2e > $O/spw4_$k.json 2>&1; done
for k in 16 64; do FZ_SLICES_PER_WARP=$k timeout 200 python tools/quick_time.py C4t2 C2c > $O/spwq_$k.log 2>&1; done
