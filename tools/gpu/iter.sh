# one build-measure iteration: GPU parity suite, memo-build phase trace, C2 launch list, quick timings, bench
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/it_tests.log 2>&1; echo "rc=$?" >> $O/it_tests.log
FZ_TRACE_CTAS=1 timeout 200 python tools/k1_trace.py C2 C3t3 C4 > $O/it_trace.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv --log-file $O/it_launch.csv python bench.py --steps 20 --warmup 10 --no-e2e --no-cpu --no-count > /dev/null 2>&1
timeout 300 python tools/quick_time.py C2 C3t3 C3t4 C4 > $O/it_qt.log 2>&1
timeout 300 python bench.py --steps 200 --no-cpu --no-e2e > $O/it_bench.json 2> $O/it_bench.err
