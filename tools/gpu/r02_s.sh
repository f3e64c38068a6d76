O=gpurun_out; T=${1:-r02s}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/quick_time.py T95 T94 T63 T74 T31 C2 C4 > $O/${T}_qt.log 2>&1
FZ_WORD_STREAM=1 timeout 300 python tools/quick_time.py T94 T63 T74 T31 > $O/${T}_qt_ws1.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
timeout 300 python tools/count_tune.py b96:g3072:t128 > $O/${T}_tune.log 2>&1
