"""Strong-scaling balance of the sharded COUNT walk on one GPU: C4 (t = 3) cut into k shards, each shard's
whole step (plan + walk) timed alone with CUDA events; reports max / mean shard time and the efficiency
T_1 / (k * max shard) that k GPUs could reach before collective and launch costs.  Each
measurement starts behind ~1 ms of GPU sleep, so the host's plan creation and kernel submission overlap device
work (as in bench.py, which enqueues its steps ahead) and the events time the device work alone."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fzinputs import C3_GENS, C3_N, C4  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402


def shard_times(g, n, t, mode, k, reps=3):
    lay = fz.Layout(g, t, n + 1, entries=(mode != "count"))
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
    memo = fz.Memo(layout=lay, workspace=ws)
    pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
    out = []
    for s in range(k):
        best = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)   # ~1 ms of GPU work first: the host's plan creation and launch
            e0.record()                    # calls are enqueued behind it and stay off the device time
            p = fz.Plan(memo, n, mode, s, k, workspace=pws)
            p.launch()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out.append(best)
    return out


fz.set_memo_cap(64 << 30)
CASES = (("C4 count t=3", C4.gens, C4.n, 3, "count"), ("C4 count t=2", C4.gens, C4.n, 2, "count"),
         ("C3 hash t=3", C3_GENS, C3_N, 3, "hash"))
want = sys.argv[1:]   # e.g. C4 -> both C4 rows
for name, g, n, t, mode in CASES:
    if want and not any(name.startswith(w) for w in want):
        continue
    t1 = shard_times(g, n, t, mode, 1)[0]
    print(f"{name}: 1 shard {t1:.3f} ms")
    for k in (2, 4, 8):
        ts = shard_times(g, n, t, mode, k)
        mx, mean = max(ts), sum(ts) / k
        print(f"  {k} shards: max {mx:.3f} ms, mean {mean:.3f} ms, max/mean {mx / mean:.3f}, "
              f"T1/(k max) = {t1 / (k * mx):.3f}")
