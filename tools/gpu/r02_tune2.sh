O=gpurun_out
timeout 1500 python tools/count_tune.py b96:g3072:t256 b96:g3072:t512 b96:g3072:t64 b64:g2048:t256 b64:g1024:t128 b128:g2048:t256 > $O/r02tune2_c4.log 2>&1
