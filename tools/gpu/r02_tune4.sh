O=gpurun_out
timeout 1500 python tools/count_tune.py b64:g1536:t128 b48:g1536:t128 b56:g1536:t128 b64:g1280:t128 b64:g1792:t128 b64:g1536:t64 b48:g1280:t128 > $O/r02tune4_c4.log 2>&1
timeout 900 python tools/count_tune.py --t2 b96:g3072:t128 b64:g1536:t128 b48:g1536:t128 > $O/r02tune4_c4t2.log 2>&1
