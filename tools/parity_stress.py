"""GPU parity stress beyond the default suite (test infrastructure: compares the CUDA path with the
oracle): seeded random and mid-size Table-1-shaped instances (fzinputs), every memo dimension t, full and
partial memos, 1-4 shards, MATERIALIZE rows element by element, COUNT (staged and unstaged) and HASH.

    python tools/parity_stress.py [first_seed] [n_seeds] [seconds]      -> one summary line per family
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fzinputs import random_instance, random_instance_mid  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 400
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 600.0
C = O.C()
stats = {"instances": 0, "checks": 0, "failures": 0}
t0 = time.time()


def check(g, n):
    want, cnt, h = C.enumerate(n, g, use_o2=True)
    want = want.reshape(-1, len(g))
    d = len(g)
    for t in range(0, d + 1):
        tops = sorted({n + 1, max(1, n // 2), max(1, (3 * n) // 4)}) if 1 <= t < d else [n + 1]
        for top in tops:
            memo = fz.memo_build(g, t, n + 1, memo_top=None if top == n + 1 else top)
            for ns in (1, 2, 3, 4):
                parts, hs, tot, ct = [], 0, 0, 0
                for s in range(ns):
                    out, rows, _ = fz.enumerate(memo, n, "materialize", shard=s, nshards=ns)
                    parts.append(out.cpu().numpy().view(np.uint32).reshape(-1, d)[:rows])
                    tot += rows
                    hs = (hs + fz.enumerate(memo, n, "hash", shard=s, nshards=ns)[2]) % (1 << 64)
                    ct += fz.enumerate(memo, n, "count", shard=s, nshards=ns)[1]
                got = np.concatenate(parts) if parts else np.zeros((0, d), np.uint32)
                ok = tot == cnt and ct == cnt and hs == h and np.array_equal(got, want)
                stats["checks"] += 1
                if not ok:
                    stats["failures"] += 1
                    print("FAIL", g, n, t, top, ns, tot, ct, cnt, hex(hs), hex(h), flush=True)
    # COUNT with the card table staged in shared memory (forced), both L >= 3 kernels (k5_runs, k5_pairs)
    os.environ["FZ_COUNT_SMEM"] = "2"
    for walk in ("runs", "pairs"):
        os.environ["FZ_COUNT_WALK"] = walk
        for t in range(0, d):
            memo = fz.memo_build(g, t, n + 1, entries=False)
            for ns in (1, 3, 7):
                ct = sum(fz.enumerate(memo, n, "count", shard=s, nshards=ns)[1] for s in range(ns))
                stats["checks"] += 1
                if ct != cnt:
                    stats["failures"] += 1
                    print("FAIL staged count", walk, g, n, t, ns, ct, cnt, flush=True)
    os.environ["FZ_COUNT_SMEM"] = ""
    os.environ["FZ_COUNT_WALK"] = ""
    # MATERIALIZE as a word stream (forced on, every t): rows element by element
    os.environ["FZ_WORD_STREAM"] = "1"
    for t in range(1, d):
        memo = fz.memo_build(g, t, n + 1)
        out, rows, _ = fz.enumerate(memo, n, "materialize")
        stats["checks"] += 1
        if rows != cnt or not np.array_equal(out.cpu().numpy().view(np.uint32).reshape(-1, d)[:rows], want):
            stats["failures"] += 1
            print("FAIL word stream", g, n, t, flush=True)
    os.environ["FZ_WORD_STREAM"] = ""


for fam, gen in (("random", random_instance), ("mid", random_instance_mid)):
    n_inst = 0
    for seed in range(first, first + count):
        if time.time() - t0 > budget:
            break
        g, n = gen(seed)[:2]
        check(tuple(g), n)
        n_inst += 1
    stats["instances"] += n_inst
    print(f"{fam}: seeds {first}..{first + n_inst - 1} checked", flush=True)
print(f"parity stress: {stats['instances']} instances, {stats['checks']} checks (every t, full + partial memos, "
      f"1-4 shards, materialize/count/hash, staged count with both kernels, word stream), {stats['failures']} failures, "
      f"{time.time() - t0:.0f} s", flush=True)
