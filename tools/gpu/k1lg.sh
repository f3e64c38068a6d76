# parity suite + memo-build timeline with the default lanes per x and forced 8/16 lanes, C2 bench
O=gpurun_out
md5sum paper_2407_20474_b200/libfz.so > $O/k1lg_md5.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/k1lg_tests.log 2>&1; echo "rc=$?" >> $O/k1lg_tests.log
for lg in "" 3 4; do echo "== FZ_SCAN_LG=$lg" >> $O/k1lg_trace.log; FZ_SCAN_LG=$lg timeout 200 python tools/k1_trace.py C2 C3t3 >> $O/k1lg_trace.log 2>&1; done
timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-count > $O/k1lg_bench.json 2>&1
