# parity suite + C2 quick timing + bench line
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/q_tests.log 2>&1; echo "rc=$?" >> $O/q_tests.log
timeout 120 python tools/quick_time.py C2 C2h > $O/q_qt.log 2>&1
timeout 300 python bench.py --steps 200 --no-cpu --no-e2e > $O/q_bench.json 2> $O/q_bench.err
