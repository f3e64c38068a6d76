O=gpurun_out
T=r02long
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
for pass in 1 2; do timeout 300 python tools/ab_time.py long C3t3 C3t2 C3t4 C2h C2 >> $O/${T}_ab.log 2>&1; done
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
