O=gpurun_out; T=${1:-r02j}
timeout 300 python tools/quick_time.py T95 T94 T63 T74 T31 > $O/${T}_auto.log 2>&1
FZ_WORD_STREAM=1 timeout 300 python tools/quick_time.py T95 T94 T63 T74 > $O/${T}_ws1.log 2>&1
FZ_WORD_STREAM=0 timeout 300 python tools/quick_time.py T95 T94 T63 T74 > $O/${T}_ws0.log 2>&1
timeout 300 python tools/fill_modes.py > $O/${T}_fill_modes.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
