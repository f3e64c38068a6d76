"""Run one configuration once (for ncu captures): python tools/prof_one.py CFG [mode]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_20474_b200 import fz  # noqa: E402
from tools.quick_time import CFG  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g, n, t, mode, *pct = CFG[name]
lay = fz.Layout(g, t, n + 1, entries=(mode != "count"), memo_top=(n * pct[0] // 100 if pct else None))
ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
memo = fz.Memo(layout=lay, workspace=ws)
pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
plan = fz.Plan(memo, n, mode, workspace=pws)
out = torch.empty((plan.rows, len(g)), dtype=torch.int32, device="cuda") if mode == "materialize" else None
for _ in range(reps):
    memo = fz.Memo(layout=lay, workspace=ws)
    plan = fz.Plan(memo, n, mode, workspace=pws)
    plan.launch(out)
torch.cuda.synchronize()
print(name, plan.result())
