O=gpurun_out
T=r02g
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python tools/shard_balance.py C4 > $O/${T}_shard_balance.log 2>&1
timeout 300 python tools/ab_time.py fin C4 C4t2 C2 T95 >> $O/${T}_ab.log 2>&1
FZ_LIB_PATH=ab/libfz_addr.so timeout 300 python tools/ab_time.py addr C4 C4t2 >> $O/${T}_ab.log 2>&1
