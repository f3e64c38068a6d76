"""C5: the 31 Table 1 scenarios on one B200: memo build vs enumerate split.

For every row (d, memo_dim, n), gens (13,37,38[,40..45])[:d], full memo top = n+1:
memo_us = fz_memo_build (K1 + K3) from a prebuilt layout, enum_us = plan + enumerate (materialize),
both CUDA-event medians of 5 runs after 2 warm-ups, beside the paper's cpu/gpu memo us and runtime ms
(RTX 3080 + Ryzen 3900X; context only).  Also runs the recommended t (fz_recommend_t).
Writes a markdown table to stdout (`--csv`: the paper's Table 1 record, as CSV)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fzinputs import TABLE1_ROWS, table1_gens  # noqa: E402
from paper_2407_20474_b200 import fz  # noqa: E402

PAPER = {}
for line in open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                              "table1.csv")):
    if line[0].isdigit():
        f = line.strip().split(",")
        PAPER[(int(f[1]), int(f[2]), int(f[3]))] = (int(f[4]), int(f[5]), int(f[6]), int(f[7]))


def timed(fn, reps=5, warm=2):
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


def run(d, t, n):
    g = table1_gens(d)
    lay = fz.Layout(g, t, n + 1)
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
    memo = fz.Memo(layout=lay, workspace=ws)
    pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
    plan = fz.Plan(memo, n, "materialize", workspace=pws)
    rows = plan.rows
    out = torch.empty((max(rows, 1), d), dtype=torch.int32, device="cuda")
    memo_us = timed(lambda: fz.Memo(layout=lay, workspace=ws))

    def en():
        p = fz.Plan(memo, n, "materialize", workspace=pws)
        p.launch(out)
    enum_us = timed(en)
    r, _ = fz.Plan(memo, n, "materialize", workspace=pws).result() if False else (rows, 0)
    return rows, memo_us, enum_us


def main_csv():
    """--csv: the paper's Table 1 record (SPEC header dim,memo_dim,element,num_results,cpu_memo_us,
    par_memo_us,runtime_ms) with this build's GPU memo build as par_memo_us and memo + enumerate as runtime_ms;
    cpu_memo_us is the single-thread CPU memo (Alg 2) recorded by `bench.py --study f4` (profiles/r02x_f4_study.jsonl;
    blank when absent); the GPU enumerate time and factorizations/s are appended."""
    import json
    cpu = {}   # recorded single-thread CPU memo times (bench.py --study f4, profiles/r02x_f4_study.jsonl)
    study = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02x_f4_study.jsonl")
    if os.path.exists(study):
        for line in open(study):
            r = json.loads(line)
            if "cpu_memo_us" in r and "t_paper" in r:
                cpu[(len(r["gens"]), r["t_paper"], r["n"])] = r["cpu_memo_us"]
    print("dim,memo_dim,element,num_results,cpu_memo_us,par_memo_us,runtime_ms,gpu_enum_us,fact_per_s")
    for d, t, n in TABLE1_ROWS:
        rows, mu, eu = run(d, t, n)
        tot = (mu + eu) / 1e3
        c = cpu.get((d, t, n))
        print(f"{d},{t},{n},{rows},{'' if c is None else f'{c:.1f}'},{mu:.1f},{tot:.4f},{eu:.1f},"
              f"{rows / tot * 1e3:.4e}", flush=True)


def main():
    if "--csv" in sys.argv:
        return main_csv()
    print("| d | t | n | rows | memo us | enum us | total ms | fact/s | t* | t* total ms | paper gpu_memo us | paper runtime ms | paper fact/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for d, t, n in TABLE1_ROWS:
        rows, mu, eu = run(d, t, n)
        tb, _ = fz.recommend_t(table1_gens(d), n, "materialize")
        if tb != t:
            _, mu2, eu2 = run(d, tb, n)
            tot2 = (mu2 + eu2) / 1e3
        else:
            tot2 = (mu + eu) / 1e3
        pr = PAPER[(d, t, n)]
        tot = (mu + eu) / 1e3
        print(f"| {d} | {t} | {n} | {rows} | {mu:.1f} | {eu:.1f} | {tot:.3f} | {rows / tot * 1e3:.3e} | {tb} | {tot2:.3f} | "
              f"{pr[2]} | {pr[3]} | {pr[0] / pr[3] * 1e3:.2e} |", flush=True)


if __name__ == "__main__":
    main()
