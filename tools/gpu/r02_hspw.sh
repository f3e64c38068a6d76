O=gpurun_out
T=r02hspw
for pass in 1 2; do
  for spw in 16 32 64 128 256; do
    FZ_SLICES_PER_WARP=$spw timeout 300 python tools/ab_time.py spw$spw C3t3 C3t2 C2h >> $O/${T}_ab.log 2>&1
  done
done
