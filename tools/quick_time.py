"""Quick CUDA-event timings of the three phases (memo build, plan, enumerate) on one config.
Usage: python tools/quick_time.py [C2|C3t2|C3t3|C4|T1]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_20474_b200 import fz  # noqa: E402

CFG = {
    "C2": ((11, 13, 17, 19), 30232, 2, "materialize"),
    "C2h": ((11, 13, 17, 19), 30232, 2, "hash"),
    "C2c": ((11, 13, 17, 19), 30232, 2, "count"),
    "C3t2": ((23, 29, 31, 37, 41, 43), 17350, 2, "hash"),
    "C3t3": ((23, 29, 31, 37, 41, 43), 17350, 3, "hash"),
    "C3t4": ((23, 29, 31, 37, 41, 43), 17350, 4, "hash"),
    "C4t2": ((97, 98, 99, 100, 101, 102, 103, 104), 40000, 2, "count"),
    "C4t4": ((97, 98, 99, 100, 101, 102, 103, 104), 40000, 4, "count"),
    "C4": ((97, 98, 99, 100, 101, 102, 103, 104), 40000, 3, "count"),
    "T1": ((13, 37, 38, 40, 41, 42, 43, 44), 2000, 4, "materialize"),
    "T95": ((13, 37, 38, 40, 41, 42, 43, 44, 45), 1500, 5, "materialize"),
    "T94": ((13, 37, 38, 40, 41, 42, 43, 44, 45), 1500, 4, "materialize"),
    "T63": ((13, 37, 38, 40, 41, 42), 5000, 3, "materialize"),
    "T31": ((13, 37, 38), 300000, 1, "materialize"),
    "T74": ((13, 37, 38, 40, 41, 42, 43), 2000, 4, "materialize"),
    "T84b": ((13, 37, 38, 40, 41, 42, 43, 44), 1500, 4, "materialize"),
    "T64": ((13, 37, 38, 40, 41, 42), 3000, 4, "materialize"),
}
# partial memo (f2): memo rows only for x < frac * n
for _f in (10, 25, 50, 75, 90):
    CFG[f"C2p{_f}"] = CFG["C2"] + (_f,)
    CFG[f"C2hp{_f}"] = CFG["C2h"] + (_f,)
CFG["C3t3p50"] = CFG["C3t3"] + (50,)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main():
    fz.set_memo_cap(64 << 30)   # C3 t=4: 30.4 GB memo (above the 8e9 default)
    names = sys.argv[1:] or ["C2"]
    for name in names:
        g, n, t, mode, *pct = CFG[name]
        mt = n * pct[0] // 100 if pct else None
        lay = fz.Layout(g, t, n + 1, entries=(mode != "count"), memo_top=mt)
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
        memo = fz.Memo(layout=lay, workspace=ws)
        pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
        plan = fz.Plan(memo, n, mode, workspace=pws)
        out = None
        if mode == "materialize":
            out = torch.empty((plan.rows, len(g)), dtype=torch.int32, device="cuda")
        for rep in range(4):
            torch.cuda.synchronize()
            e0 = ev()
            memo = fz.Memo(layout=lay, workspace=ws)
            e1 = ev()
            plan = fz.Plan(memo, n, mode, workspace=pws)
            e2 = ev()
            plan.launch(out)
            e3 = ev()
            torch.cuda.synchronize()
            rows, h = plan.result()
            mb, pl, en = e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3)
            extra = ""
            if mode == "materialize":
                extra = f" write {rows * len(g) * 4 / en / 1e6:.1f} GB/s"
            print(f"{name} rep{rep}: memo {mb*1e3:.1f} us (mode {memo.info['fill_mode']}, batches "
                  f"{memo.info['batches']}, entries {memo.info['entries']}), plan {pl*1e3:.1f} us "
                  f"({plan.nslices} slices), enum {en*1e3:.1f} us, rows {rows} hash {h:#x} "
                  f"-> {rows / ((mb + pl + en) / 1e3):.3e} fact/s{extra}", flush=True)
        del out


if __name__ == "__main__":
    main()
