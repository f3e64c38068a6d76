O=gpurun_out
timeout 1500 python tools/count_tune.py b96:g3072:t128 b128:g3072:t128 b128:g6144:t128 b192:g6144:t128 b64:g6144:t128 b192:g12288:t128 b256:g8192:t128 > $O/r02tune_c4.log 2>&1
