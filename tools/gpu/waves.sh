# K5 materialize on a multi-wave grid (FZ_K5_WAVES): parity subset + bench
O=gpurun_out
md5sum paper_2407_20474_b200/libfz.so > $O/w_md5.txt
FZ_K5_WAVES=8 timeout 600 python -m pytest tests -m gpu -x -q -k "c2_full or mid_sharded or random_small or table1_rows or partial" > $O/w_tests.log 2>&1; echo "rc=$?" >> $O/w_tests.log
for w in 0 2 4 8 16; do FZ_K5_WAVES=$w timeout 200 python bench.py --steps 200 --no-cpu --no-e2e --no-count > $O/w_$w.json 2>&1; done
