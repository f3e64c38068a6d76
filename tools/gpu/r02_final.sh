O=gpurun_out
T=r02y
python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/table1_bench.py --csv > $O/${T}_table1.csv 2>&1
timeout 300 python bench.py --steps 50 > $O/${T}_bench.json 2> $O/${T}_bench.err
