O=gpurun_out
for G in 148 1 2 8 32; do FZ_K1_GRID=$G timeout 300 python tools/table1_bench.py --csv > $O/r02k1_grid$G.csv 2>&1; done
for G in 148 1 4 16; do FZ_K1_GRID=$G timeout 300 python tools/quick_time.py C2 C4 > $O/r02k1_qt$G.log 2>&1; done
