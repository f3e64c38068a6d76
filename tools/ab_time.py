"""A/B timing of the walk kernel (K5) of one config: median / min of R CUDA-event timed plan.launch calls,
rows and hash printed for a correctness glance.  The library is the one FZ_LIB_PATH names (default build
otherwise).  Usage: FZ_LIB_PATH=ab/libfz_X.so python tools/ab_time.py TAG C4 T95 ..."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_20474_b200 import fz  # noqa: E402
from tools.quick_time import CFG  # noqa: E402


def main():
    fz.set_memo_cap(64 << 30)
    tag, names = sys.argv[1], sys.argv[2:]
    for name in names:
        g, n, t, mode, *pct = CFG[name]
        lay = fz.Layout(g, t, n + 1, entries=(mode != "count"))
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
        memo = fz.Memo(layout=lay, workspace=ws)
        pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
        plan = fz.Plan(memo, n, mode, workspace=pws)
        out = torch.empty((plan.rows, len(g)), dtype=torch.int32, device="cuda") if mode == "materialize" else None
        reps = 5 if name.startswith(("C3", "C4t2")) else 15
        ts = []
        for _ in range(reps):
            plan = fz.Plan(memo, n, mode, workspace=pws)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.launch(out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        rows, h = plan.result()
        print(f"{tag} {name}: K5 median {statistics.median(ts):.1f} us min {min(ts):.1f} us, rows {rows} "
              f"hash {h:#x}", flush=True)
        del out


if __name__ == "__main__":
    main()
