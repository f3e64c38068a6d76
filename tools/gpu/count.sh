# parity suite + COUNT timings
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/c_tests.log 2>&1; echo "rc=$?" >> $O/c_tests.log
timeout 200 python tools/quick_time.py C4 C4t2 C2c > $O/c_qt.log 2>&1
timeout 300 python bench.py --config C4 --steps 20 --no-cpu --no-e2e > $O/c_bench.json 2> $O/c_bench.err
