"""COUNT pair-walk cost-model sweep on one GPU: for each setting (beta = FZ_COUNT_RUN_COST, gamma =
FZ_COUNT_OUTER_COST, tail = FZ_GSS_TAIL) time C4 (t = 3, and t = 2 with --t2) whole and cut into 4 and 8
shards (plan + walk of each shard alone, CUDA events, best of 3).
Usage: python tools/count_tune.py [--t2] b32:g0:t128 b64:g256:t128 ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fzinputs import C4  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402


def shard_ms(memo, n, k, s, pws, reps=3):
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)   # the host's plan / launch calls are enqueued behind ~1 ms of GPU work
        e0.record()
        p = fz.Plan(memo, n, "count", s, k, workspace=pws)
        p.launch()
        e1.record()
        torch.cuda.synchronize()
        best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
    return best, p.result()[0]


args = [a for a in sys.argv[1:] if not a.startswith("--")]
ts = [2] if "--t2" in sys.argv else [3]
for t in ts:
    for spec in args or ["b32:g0:t128"]:
        kv = {x[0]: x[1:] for x in spec.split(":")}
        os.environ["FZ_COUNT_RUN_COST"] = kv.get("b", "32")
        os.environ["FZ_COUNT_OUTER_COST"] = kv.get("g", "0")
        os.environ["FZ_GSS_TAIL"] = kv.get("t", "128")
        lay = fz.Layout(C4.gens, t, C4.n + 1, entries=False)
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
        memo = fz.Memo(layout=lay, workspace=ws)
        pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
        t1, r1 = shard_ms(memo, C4.n, 1, 0, pws)
        line = f"t={t} {spec}: T1 {t1:.3f} ms rows {r1}"
        for k in (2, 4, 8):
            res = [shard_ms(memo, C4.n, k, s, pws) for s in range(k)]
            tk = [x[0] for x in res]
            assert sum(x[1] for x in res) == r1
            mx, mean = max(tk), sum(tk) / k
            line += f" | k={k}: max {mx:.3f} mean {mean:.3f} eff {t1 / (k * mx):.3f}"
        print(line, flush=True)
