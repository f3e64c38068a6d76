# K5 materialize with and without its output stores (FZ_K5_DIAG=1), and the pure streaming-fill ceiling
O=gpurun_out
timeout 120 python tools/quick_time.py C2 > $O/k5d_base.log 2>&1
FZ_K5_DIAG=1 timeout 120 python tools/quick_time.py C2 > $O/k5d_nostore.log 2>&1
timeout 120 ./tools/micro/write_bw > $O/k5d_wbw.log 2>&1
