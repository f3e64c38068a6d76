O=gpurun_out
T=r02z
md5sum paper_2407_20474_b200/libfz.so > $O/${T}_md5.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 300 python bench.py --config C4 --steps 20 --no-cpu > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err
