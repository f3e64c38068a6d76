"""C1: Z(m; 6,9,20) for every m <= 1000 on one B200, two routes.

(a) full DP table (t = d = 3): ONE memo build produces every list -- the table
    of Alg 2/3 is exactly C1's output (162 781 rows);
(b) memo t = 2 (top 1001) + 1001 separate plan + enumerate calls (latency-bound).
CUDA-event medians; prints a markdown table."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fzinputs import C1_GENS, C1_MAX_N  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main():
    g, N = C1_GENS, C1_MAX_N
    lay = fz.Layout(g, len(g), N + 1)
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(7):
        torch.cuda.synchronize()
        a = ev()
        fz.Memo(layout=lay, workspace=ws)
        b = ev()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ta = sorted(ts)[3]
    rows_a = lay.info["entries"]

    lay2 = fz.Layout(g, 2, N + 1)
    ws2 = torch.empty(lay2.workspace_bytes, dtype=torch.uint8, device="cuda")
    out = torch.empty((600, 3), dtype=torch.int32, device="cuda")
    pws = torch.empty(256, dtype=torch.uint8, device="cuda")
    tb = []
    for _ in range(3):
        torch.cuda.synchronize()
        a = ev()
        m = fz.Memo(layout=lay2, workspace=ws2)
        for n in range(N + 1):
            fz.Plan(m, n, "materialize", workspace=pws).launch(out)
        b = ev()
        torch.cuda.synchronize()
        tb.append(a.elapsed_time(b) * 1e3)
    tbm = sorted(tb)[1]
    print("| route | launches | time us | rows | fact/s |")
    print("|---|---|---|---|---|")
    print(f"| (a) full table t=3, one memo build | {2 + 2 * 2} | {ta:.1f} | {rows_a} | {rows_a / ta * 1e6:.3e} |")
    print(f"| (b) memo t=2 + 1001 x (plan + enumerate) | ~{2 * (N + 1) + 4} | {tbm:.1f} | 162781 | {162781 / tbm * 1e6:.3e} |")


if __name__ == "__main__":
    main()
