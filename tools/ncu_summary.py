"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.md>     # --metrics gpu__time_duration.sum list
  python tools/ncu_summary.py full <report.ncu-rep | raw.csv> <out.md> [key]  # --set full capture (one or more kernels)

`full` also merges {key: {dram_bytes_per_launch, warp_inst_per_launch, ...}} into profiles/k5_counters.json.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0]
            if name not in per:
                order.append(name)
            per[name].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in per.values())
    lines = [f"# Launch list: `{os.path.basename(path)}`", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised launches:",
             "compare shares, not absolute times).", "",
             "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k in order:
        v = per[k]
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, key=None):
    if rep.endswith(".csv"):   # `ncu -i X.ncu-rep --page raw --csv` exported on the GPU box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rd[0], rd[1], rd[2:]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "smsp__inst_executed_op_shared_ld.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full: `{os.path.basename(rep)}`", ""]
    summ = {}
    for r in data:
        name = r[idx["Kernel Name"]][:90]
        lines.append(f"## `{name}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for w in want:
            if w in idx:
                lines.append(f"| {w} | {r[idx[w]]} | {units[idx[w]]} |")
                vals[w] = (r[idx[w]], units[idx[w]])
        lines.append("")
        summ[name] = vals
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if key:
        def tobytes(v):
            x, u = v
            x = float(x.replace(",", ""))
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        k5 = [v for n, v in summ.items() if any(k in n for k in ("k5_walk", "k5_runs", "k5_pairs"))]
        if k5:
            v = k5[0]
            dram = tobytes(v["dram__bytes_read.sum"]) + tobytes(v["dram__bytes_write.sum"])
            # bench.py reads profiles/k5_counters.json (per-launch DRAM bytes and warp instructions of each
            # leg's dominant kernel at the kernel version captured)
            p = os.path.join(ROOT, "profiles", "k5_counters.json")
            cur = json.load(open(p)) if os.path.exists(p) else {}
            cur[key] = {"dram_bytes_per_launch": dram, "dram_read": tobytes(v["dram__bytes_read.sum"]),
                        "dram_write": tobytes(v["dram__bytes_write.sum"]),
                        "warp_inst_per_launch": float(v["smsp__inst_executed.sum"][0].replace(",", "")),
                        "duration_ns": float(v["gpu__time_duration.sum"][0].replace(",", "")) *
                        {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(
                            v["gpu__time_duration.sum"][1], 1),
                        "source": os.path.basename(out)}
            json.dump(cur, open(p, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
