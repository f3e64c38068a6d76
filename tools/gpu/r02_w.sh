O=gpurun_out; T=${1:-r02w}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/quick_time.py T95 T63 T74 C4 C2 > $O/${T}_qt.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
