# re-entry check of HEAD: GPU parity suite, quick timings of every config, C4 / C3 / T95 bench-like numbers
O=gpurun_out
T=${1:-r02h}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > $O/${T}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 400 python tools/quick_time.py C2 C2h C2c C3t2 C3t3 C4 T1 T95 T94 T63 > $O/${T}_quick_time.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
