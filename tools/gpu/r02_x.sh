O=gpurun_out; T=${1:-r02x}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/quick_time.py T95 T94 T63 T74 C2 C2h C3t3 C3t2 C4 > $O/${T}_qt.log 2>&1
FZ_ROW_GSS=0 timeout 300 python tools/quick_time.py T95 T94 T63 T74 C2 C2h C3t3 > $O/${T}_qt_nogss.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
timeout 300 python tools/shard_balance.py C3 > $O/${T}_sb_c3.log 2>&1
