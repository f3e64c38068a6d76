O=gpurun_out; T=${1:-r02y}
timeout 900 python -m pytest tests -m gpu -x -q -k "large_materialize or c4_count or c2_full or run_host" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/quick_time.py T95 T94 T63 T74 C2 C2h C3t3 C3t2 C4 C4t2 > $O/${T}_qt.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
