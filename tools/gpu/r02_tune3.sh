O=gpurun_out
timeout 1500 python tools/count_tune.py b96:g3072:t128 b64:g2048:t256 b64:g2048:t64 b48:g2048:t128 b64:g1536:t128 b80:g2048:t128 b64:g2560:t128 b64:g2048:t128 > $O/r02tune3_c4.log 2>&1
