"""SURVEY §8(f) f1 schedule timing (the DP can be parallelised elementwise -- batches of
b <= min(tail g) consecutive elements, each batch's factorizations in parallel -- or factorizationwise, "or
both"): memo build time of each copy-increment schedule (fill modes 1-5, fz_set_fill_mode), CUDA-event
median of 7 builds after 2 warm-ups, on C1 (t = 2 memo and the t = d full table), C2's memo and Table 1
memos.  Every mode builds the same rows (tests/test_gpu_parity.py::test_memo_rows_vs_alg2).
Writes a markdown table to stdout."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fzinputs import table1_gens  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402

MODES = {1: "elementwise batches of min(tail g), one CTA, smem ring (the paper's schedule)",
         2: "same through L2", 3: "elementwise batches over the whole grid (grid barrier per batch)",
         4: "per tail dimension, residue chains stepped in order",
         5: "per tail dimension, chains in scan form (default)"}
CASES = [("C1 t=2", (6, 9, 20), 2, 1001), ("C1 t=3 (full table, f1)", (6, 9, 20), 3, 1001),
         ("C2 t=2", (11, 13, 17, 19), 2, 30233),
         ("T1 (6,4,3000)", table1_gens(6), 4, 3001), ("T1 (8,4,2000)", table1_gens(8), 4, 2001),
         ("T1 (9,5,1500)", table1_gens(9), 5, 1501), ("T1 (5,3,5000)", table1_gens(5), 3, 5001)]


def timed(fn, reps=7, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[len(ts) // 2]


print("| memo | entries | batches | " + " | ".join(f"mode {m} us" for m in MODES) + " |")
print("|---|---|---|" + "---|" * len(MODES))
for name, g, t, top in CASES:
    cells, info = [], None
    for mode in MODES:
        fz.set_fill_mode(mode)
        lay = fz.Layout(g, t, top)
        if lay.info["fill_mode"] != mode:       # the schedule does not fit this memo (e.g. ring > smem)
            cells.append("n/a")
            continue
        info = lay.info
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
        cells.append(f"{timed(lambda: fz.Memo(layout=lay, workspace=ws)):.1f}")
        del ws
    fz.set_fill_mode(0)
    print(f"| {name} | {info['entries'] if info else '-'} | {info['batches'] if info else '-'} | " + " | ".join(cells) + " |")
print()
for m, s in MODES.items():
    print(f"- mode {m}: {s}")
