"""Small GPU workload for compute-sanitizer: every fill mode, every K5 mode, t = 0 / d, shards."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402

C = O.C()
cases = [((13, 37, 38, 40), 800, 2), ((6, 9, 20), 300, 2), ((3, 5, 8, 11), 200, 3), ((7, 7, 3), 150, 1),
         ((13, 37, 38, 40, 41), 600, 3), ((5,), 40, 0), ((6, 9, 20), 120, 3)]
bad = 0
for fill in (0, 1, 2, 3, 4, 5):
    fz.set_fill_mode(fill)
    for g, n, t in cases:
        memo = fz.memo_build(g, t, n + 1)
        want, cnt, h = C.enumerate(n, g)
        for ns in (1, 3):
            got, hs = [], 0
            for s in range(ns):
                out, r, _ = fz.enumerate(memo, n, "materialize", shard=s, nshards=ns)
                got.append(out.cpu().numpy().view(np.uint32).reshape(-1, len(g))[:r])
                hs = (hs + fz.enumerate(memo, n, "hash", shard=s, nshards=ns)[2]) % (1 << 64)
            ok = np.array_equal(np.concatenate(got), want.reshape(-1, len(g))) and hs == h
            ok = ok and fz.enumerate(memo, n, "count")[1] == cnt
            bad += (not ok)
fz.set_fill_mode(0)
# staged COUNT walks forced on small instances: the outer-prefix walk (L >= 3) and the run-per-lane walk (L = 2)
os.environ["FZ_COUNT_SMEM"] = "2"
for g, n, t in [((13, 37, 38, 40, 41), 600, 1), ((3, 5, 8, 11), 200, 1), ((3, 5, 8, 11), 200, 2),
                ((13, 37, 38, 40, 41), 600, 2)]:
    memo = fz.memo_build(g, t, n + 1, entries=False)
    cnt = C.gf_count(n, g)
    for ns in (1, 3):
        bad += sum(fz.enumerate(memo, n, "count", shard=s, nshards=ns)[1] for s in range(ns)) != cnt
for walk in ("runs", "pairs"):   # both COUNT kernels of L >= 3
    os.environ["FZ_COUNT_WALK"] = walk
    for g, n, t in [((13, 37, 38, 40, 41), 600, 2), ((3, 5, 8, 11, 13), 200, 1), ((97, 98, 99, 100, 101), 900, 2)]:
        memo = fz.memo_build(g, t, n + 1, entries=False)
        cnt = C.gf_count(n, g)
        for ns in (1, 3):
            bad += sum(fz.enumerate(memo, n, "count", shard=s, nshards=ns)[1] for s in range(ns)) != cnt
os.environ["FZ_COUNT_SMEM"] = ""
os.environ["FZ_COUNT_WALK"] = ""
# the MATERIALIZE word stream (odd d, long rounds) and the end-to-end output ring (tiny slots: many chunks)
os.environ["FZ_WORD_STREAM"] = "1"
for g, n, t in [((13, 37, 38, 40, 41), 900, 3), ((13, 37, 38, 40, 41, 42, 43, 44, 45), 600, 5)]:
    memo = fz.memo_build(g, t, n + 1)
    want, cnt, h = C.enumerate(n, g)
    out, r, _ = fz.enumerate(memo, n, "materialize")
    bad += not np.array_equal(out.cpu().numpy().view(np.uint32).reshape(-1, len(g))[:r], want.reshape(-1, len(g)))
os.environ["FZ_WORD_STREAM"] = ""
import torch  # noqa: E402
g, n, t = (13, 37, 38, 40), 3000, 2
want, cnt, h = C.enumerate(n, g)
host = torch.empty((cnt, len(g)), dtype=torch.int32).pin_memory()
r, _ = fz.run_host(g, t, n, "materialize", host, ring_bytes=4096)
bad += (r != cnt) or not np.array_equal(host.numpy().view(np.uint32), want.reshape(-1, len(g)))
print("sanitize subset:", "OK" if bad == 0 else f"{bad} FAILURES")
