O=gpurun_out; T=${1:-r02i}
timeout 300 python tools/quick_time.py T95 T63 T31 T74 C2 T1 > $O/${T}_ws1.log 2>&1
FZ_WORD_STREAM=0 timeout 300 python tools/quick_time.py T95 T63 T31 T74 > $O/${T}_ws0.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
timeout 300 python tools/fill_modes.py > $O/${T}_fill_modes.log 2>&1
timeout 400 python bench.py --steps 50 --no-cpu > $O/${T}_bench.json 2> $O/${T}_bench.err
