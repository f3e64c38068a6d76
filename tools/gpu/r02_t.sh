O=gpurun_out; T=${1:-r02t}
timeout 600 python -m pytest tests -m gpu -x -q -k "count or device_plan or random_small or mid_sharded" > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 300 python tools/count_tune.py b96:g3072:t128 b96:g3072:t64 > $O/${T}_tune.log 2>&1
timeout 300 python tools/count_tune.py --t2 b96:g3072:t128 > $O/${T}_tune_t2.log 2>&1
timeout 900 python tools/parity_stress.py 5000 400 720 > $O/${T}_stress.log 2>&1
