"""bench.py -- factorizations/sec of the whole hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--config C2|C4]

A step is one pass of the whole hot path over one problem: memo build on the
GPU (count pass K1 + copy-increment recurrence K3), device-side shard plan K4, enumeration K5 and, when
one problem is cut into shards over N > 1 ranks, the NCCL all_reduce of the {rows, hash} accumulators
(A10).  The A1 host layout (validation + sizing, like an FFT plan) is made once per configuration,
outside the timed region.

Headline workload:
  N = 1: BASELINE.json configs[1] (C2: Z(30232; 11,13,17,19), 100 000 681 rows materialized).
  N > 1: ONE count problem cut into N shards (C4: Z(40000; 97..104), t = 3, 3.36e12 rows; BASELINE
         configs[3], the north-star multi-GPU target) -> "scaling": "strong".  The same line carries the
         other legs as extra keys ("legs"): C2 materialize row-sharded (strong) and the C2 batch of N
         independent elements (weak), so each workload can be compared across N.
  --config C4 (or C2) forces the headline workload at any N.
At N = 1 the line also carries count_mode (C2, C4 t=3) and hash_mode (C3 t=3) legs, each with a roofline.

`python bench.py --gpus N` without torchrun spawns the N ranks itself (torch.distributed.run, one process
per GPU, NCCL); with fewer visible GPUs than N the ranks share them over gloo, and the line says so.

`--impl reference` times the CPU oracle (oracle/, the plain nested-loop definition) on this host's cores
on a bounded sample of the same workload (there is no reference program to install: the reference is a
paper).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factorizations/sec at 1/2/4/8 B200 (materialize + count); % of HBM-write roofline"
UNIT = "factorizations/s"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def workload(name: str, rank: int, world: int):
    """The bench workloads (fixed tuples from fzinputs, BASELINE.json configs)."""
    from fzinputs import C2, C4

    if name == "C2":        # configs[1]: one element materialized (N = 1), or row-sharded over the ranks
        return dict(name="C2", gens=C2.gens, n=C2.n, t=C2.t, mode="materialize", shard=rank, nshards=world,
                    scaling="strong" if world > 1 else "weak")
    if name == "C2batch":   # N independent elements, one per rank (n_r = 30232 - r)
        return dict(name="C2batch", gens=C2.gens, n=C2.n - rank, t=C2.t, mode="materialize", shard=0, nshards=1,
                    scaling="weak")
    if name == "C4":        # configs[3]: one count problem cut into N shards
        return dict(name="C4", gens=C4.gens, n=C4.n, t=C4.t, mode="count", shard=rank, nshards=world,
                    scaling="strong")
    if name == "C4t2":
        return dict(name="C4t2", gens=C4.gens, n=C4.n, t=2, mode="count", shard=rank, nshards=world,
                    scaling="strong")
    raise SystemExit(f"unknown workload {name}")


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _profile_counters():
    """Per-launch counters captured once with ncu (profiles/k5_counters.json): DRAM bytes and warp
    instructions of each leg's dominant kernel at the current kernel version."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "k5_counters.json")))
    except Exception:
        return {}


def leading_prefixes(g, n: int, L: int) -> int:
    """Leading prefixes (a_1..a_L) with phi <= n = sum_{x<=n} |Z(x; g_1..g_L)| (coin-change counts;
    measurement bookkeeping for the COUNT roofline, not part of the product path)."""
    import numpy as np

    c = np.zeros(n + 1, dtype=np.int64)
    c[0] = 1
    for gi in g[:L]:
        for r in range(min(gi, n + 1)):
            c[r::gi] = np.cumsum(c[r::gi])
    return int(c.sum())


def roofline(W, plan, k5_ms: float, rows_local: int, sm_max_mhz, props, world: int):
    """Roofline of the leg's dominant kernel (K5): algorithmic units per launch / its CUDA-event time.
    MATERIALIZE: HBM bytes written (4 d per row).  COUNT: card lookups (one per leading prefix, SURVEY
    §8(d)) against the shared-memory crossbar, 128 B/clk/SM (B300_MICROARCH.md LDS/STS) / bytes per card.
    HASH: issue slots -- the kernel's ncu warp-instruction count (profiles/k5_counters.json) against
    SMs x 4 SMSPs x 1 instr/clk."""
    g, n, t, mode = W["gens"], W["n"], W["t"], W["mode"]
    d = len(g)
    peaks = _peaks()
    clk = (sm_max_mhz or peaks.get("sm_max_mhz") or 1965) * 1e6
    sms = props.multi_processor_count
    walk, card_bytes = plan.walk()
    counters = _profile_counters().get(W["name"], {})
    if mode == "materialize":
        alg = rows_local * d * 4
        peak = peaks.get("hbm_gbs")
        r = {"kernel": f"k5_walk<{d},{t},materialize>", "bound": "hbm", "achieved": alg / (k5_ms / 1e3) / 1e9,
             "peak": peak if peak else 6650.0,
             "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peak else "fallback (B200_PROFILING.md)",
             "unit": "GB/s", "algorithmic_bytes_per_launch": alg,
             "derivation": "4 d bytes per output row (one 16-B store per row at d = 4) / K5 event time"}
    elif mode == "count":
        U = leading_prefixes(g, n, d - t)
        units = U / W["nshards"]
        peak = sms * 128 / card_bytes * clk
        kname = {"count_staged": "k5_runs", "count_pairs": "k5_pairs"}.get(walk)
        r = {"kernel": f"{kname}<{d},{t},{'u8' if card_bytes == 1 else 'u16'}>" if kname
             else f"k5_walk<{d},{t},count>", "bound": "smem",
             "achieved": units / (k5_ms / 1e3), "peak": peak, "unit": "card lookups/s",
             "peak_source": (f"derived: {sms} SMs x 128 B/clk shared-memory crossbar (B300_MICROARCH.md LDS/STS) / "
                             f"{card_bytes} B per card x {clk / 1e6:.0f} MHz"),
             "algorithmic_units_per_launch": units,
             "derivation": "one card lookup per leading prefix (a_1..a_{d-t}), SURVEY §8(d); / K5 event time"}
        if W["nshards"] > 1:
            r["units_note"] = "mean lookups per shard (the cut balances modelled cost, not lookups)"
    else:
        inst = counters.get("warp_inst_per_launch")
        peak = sms * 4 * clk
        r = {"kernel": f"k5_walk<{d},{t},hash>", "bound": "issue", "unit": "warp instructions/s", "peak": peak,
             "peak_source": f"derived: {sms} SMs x 4 SMSPs x 1 warp instruction/clk x {clk / 1e6:.0f} MHz",
             "achieved": (inst / (k5_ms / 1e3)) if inst else None,
             "algorithmic_units_per_launch": inst,
             "derivation": ("warp instructions per launch from ncu (smsp__inst_executed.sum, "
                            "profiles/k5_counters.json) / K5 event time")}
    r["frac"] = (r["achieved"] / r["peak"]) if r.get("achieved") else None
    r["traffic"] = counters.get("dram_bytes_per_launch")
    r["k5_ms"] = k5_ms
    r["walk"] = walk
    return r


# ------------------------------------------------------------------ native arm
def measure(W, steps: int, warmup: int, rank: int, world: int, dev, sampler=None):
    """Time `steps` whole steps of workload W on this rank (barrier + synchronize on both sides, CUDA
    events on the launching stream, max over ranks).  Returns a dict."""
    import torch
    import torch.distributed as dist

    from paper_2407_20474_b200 import fz

    g, n, t, mode = W["gens"], W["n"], W["t"], W["mode"]
    lay = fz.Layout(g, t, n + 1, entries=mode != "count")          # A1 (host, once)
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device=dev)
    memo = fz.Memo(layout=lay, workspace=ws)
    pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device=dev)
    plan = fz.Plan(memo, n, mode, W["shard"], W["nshards"], workspace=pws)
    rows_local = plan.rows
    out = (torch.empty((max(rows_local, 1), len(g)), dtype=torch.int32, device=dev)
           if mode == "materialize" else None)
    stream = torch.cuda.current_stream()
    collective = world > 1 and W["scaling"] == "strong"

    def step(ev=None):
        m = fz.Memo(layout=lay, workspace=ws)                               # K1 + K3
        p = fz.Plan(m, n, mode, W["shard"], W["nshards"], workspace=pws)    # K4
        if ev is not None:
            ev[0].record(stream)
        p.launch(out)                                                       # K5
        if ev is not None:
            ev[1].record(stream)
        if collective:   # A10: {rows, hash} of the shards of ONE problem, NCCL, straight from the plan header
            dist.all_reduce(p.result_tensor(), op=dist.ReduceOp.SUM)
        return m, p

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    m0, p0 = step()
    torch.cuda.synchronize()
    r_step, h_step = p0.result()
    if not collective:
        assert r_step == rows_local, (r_step, rows_local)
    if world > 1 and not collective:   # rows of the whole batch, once, outside the timed region
        rt = torch.tensor([r_step], dtype=torch.float64, device=dev)
        dist.all_reduce(rt, op=dist.ReduceOp.SUM)
        r_step = int(rt.item())
    k5_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches0 = fz.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        e0.record(stream)
        keep = [step(k5_ev[k]) for k in range(steps)]
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = fz.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    k5_ms = sum(a.elapsed_time(b) for a, b in k5_ev) / steps
    tt = torch.tensor([ms, k5_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_max, k5_max = float(tt[0]), float(tt[1])
    del keep
    return {"value": float(r_step) * steps / (ms_max / 1e3), "ms_per_step": ms_max / steps, "rows_step": int(r_step),
            "rows_local": int(rows_local), "hash_step": int(h_step), "k5_ms": k5_ms, "k5_ms_max_rank": k5_max,
            "launches": launches, "plan": p0, "fill_mode": lay.info["fill_mode"]}


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _leg_line(W, r, props, clk, world):
    d = {"workload": f"{W['name']}: Z({W['n']}; {','.join(map(str, W['gens']))}) {W['mode']}, t={W['t']}",
         "value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"], "rows": r["rows_step"],
         "scaling": W["scaling"], "shards": W["nshards"]}
    d["roofline"] = roofline(W, r["plan"], r["k5_ms"], r["rows_local"], clk, props, world)
    return d


def run_native(args, rank, world, local_rank, backend):
    import torch

    dev = torch.device("cuda", local_rank)
    props = torch.cuda.get_device_properties(dev)
    head_name = args.config or ("C2" if world == 1 else "C4")
    W = workload(head_name, rank, world)
    sampler = ClockSampler(local_rank)
    r = measure(W, args.steps, args.warmup, rank, world, dev, sampler)
    clocks = sampler.summary()
    res = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": W["scaling"], "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (fixed generator tuples; no datasets)",
        "config": {"workload": f"{W['name']}: Z(n; {','.join(map(str, W['gens']))}) {W['mode']}, memo t={W['t']}, "
                               f"top=n+1" + (f", cut into {world} shards (one problem)" if W["nshards"] > 1 else ""),
                   "n": W["n"], "gens": list(W["gens"]), "t": W["t"], "mode": W["mode"],
                   "rows_per_step": r["rows_step"], "rows_this_rank": r["rows_local"], "fill_mode": r["fill_mode"],
                   "l2": ("each step writes its output (1.6 GB at N = 1, > 126 MB L2), flushing L2 between steps"
                          if W["mode"] == "materialize" else
                          "count mode: the card image is staged in shared memory each launch; tables L2-resident "
                          "by design (no output)"),
                   "parallelism": f"{'shard' if W['scaling'] == 'strong' and world > 1 else 'batch'}{world}"},
        "gpu_launches": r["launches"],
        "roofline": roofline(W, r["plan"], r["k5_ms"], r["rows_local"], clocks.get("sm_max_mhz"), props, world),
        "clocks": clocks,
    }
    if world > 1:
        res["config"]["backend"] = backend
        res["config"]["collective"] = ("all_reduce(SUM) of the 16-byte {rows, hash} shard accumulators each step "
                                       f"over {backend}" if W["scaling"] == "strong" else
                                       "none in the data path (independent elements per rank)")
    return res, W, r


def native_legs(args, rank, world, local_rank, head):
    """The other workloads on the same ranks (each timed like the headline): at N = 1 count C2 / C4 and hash
    C3; at N > 1 C2 materialize row-sharded (strong) and the C2 batch (weak), plus C4 if not the headline."""
    import torch

    dev = torch.device("cuda", local_rank)
    props = torch.cuda.get_device_properties(dev)
    legs = {}
    if world == 1:
        names = ["C4", "C2count"] if head != "C4" else ["C2"]
    else:
        names = [x for x in ("C2", "C2batch", "C4") if x != head]
    for name in names:
        if name == "C2count":
            W = workload("C2", rank, world)
            W = dict(W, name="C2count", mode="count")
        else:
            W = workload(name, rank, world)
        steps = 20 if W["mode"] == "count" and W["name"].startswith("C4") else 50
        r = measure(W, steps, 3, rank, world, dev)
        legs[W["name"]] = _leg_line(W, r, props, None, world)
    if world == 1 and not args.no_hash:
        legs["C3hash"] = hash_leg(dev, props)
    return legs


def hash_leg(dev, props):
    """Hash mode on BASELINE.json configs[2] (C3: Z(17350; 23,29,31,37,41,43), 1.0e10 rows, t = 3): whole
    step (memo build + plan + the HASH walk), CUDA-event timed; (count, H) compared with the known answer in
    tests/golden/hash_kats.csv."""
    from fzinputs import C3_GENS, C3_N

    W = dict(name="C3hash", gens=C3_GENS, n=C3_N, t=3, mode="hash", shard=0, nshards=1, scaling="weak")
    kat = None
    for line in open(os.path.join(ROOT, "tests", "golden", "hash_kats.csv")):
        f = line.strip().split(",")
        if len(f) >= 4 and f[0] == ";".join(map(str, C3_GENS)) and f[1] == str(C3_N):
            kat = (int(f[2]), int(f[3], 16))
    r = measure(W, 3, 3, 0, 1, dev)
    d = _leg_line(W, r, props, None, 1)
    d["hash"] = f"{r['hash_step']:#018x}"
    d["kat_match"] = kat == (r["rows_step"], r["hash_step"])
    return d


def run_e2e(args, W, rank, world, local_rank):
    """Same metric end to end through the public API from HOST buffers, on every rank; the timed region
    (barrier-bracketed, max over ranks) holds each step's H2D of the generator tuple and D2H of the result.
    MATERIALIZE: fz_run_host, rows streamed through the 64 MB device output ring into pinned host memory.
    COUNT (one problem cut into shards): this rank's shard through Layout/Memo/Plan with the all_reduce
    of {rows, hash}, then the 16-byte D2H read of the global result."""
    import torch
    import torch.distributed as dist

    from paper_2407_20474_b200 import fz

    g, n, t, mode = W["gens"], W["n"], W["t"], W["mode"]
    d = len(g)
    dev = torch.device("cuda", local_rank)
    steps = max(1, min(args.steps, 3))
    collective = world > 1 and W["scaling"] == "strong"
    if mode == "materialize":
        # each rank streams its own element (the batch) or its shard's rows (row-sharded, via the same call on
        # the whole element would repeat work): the e2e leg of materialize is the per-rank element
        nn = n - rank if world > 1 else n
        ws = torch.empty(fz.run_workspace_bytes(g, t, nn, mode), dtype=torch.uint8, device=dev)
        lay = fz.Layout(g, t, nn + 1, entries=True)
        rows = lay.shard_rows(nn, mode, 1)[1][0]
        host = torch.empty((rows, d), dtype=torch.int32).pin_memory()

        def one():
            return fz.run_host(g, t, nn, mode, host, workspace=ws)[0]
    else:
        lay = fz.Layout(g, t, n + 1, entries=False)
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device=dev)
        pws = None
        g_host = torch.tensor(list(g), dtype=torch.int32).pin_memory()
        g_dev = torch.empty_like(g_host, device=dev)

        def one():
            nonlocal pws
            g_dev.copy_(g_host, non_blocking=True)          # the step's input, H2D
            m = fz.Memo(layout=lay, workspace=ws)
            if pws is None:
                pws = torch.empty(fz.plan_workspace_bytes(m), dtype=torch.uint8, device=dev)
            p = fz.Plan(m, n, mode, W["shard"], W["nshards"], workspace=pws)
            p.launch()
            if collective:
                dist.all_reduce(p.result_tensor(), op=dist.ReduceOp.SUM)
            return p.result()[0]                            # D2H of {rows, hash}
    one()                                                   # warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    tot = 0
    for _ in range(steps):
        tot += one()
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t0, float(tot)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        mx = el.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = el.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        el_s = float(mx[0])
        tot = float(el[1]) if collective else float(sm[1])   # strong: all_reduced already
    else:
        el_s = float(el[0])
    local_rows = int(el[1].item()) // steps
    return {"value": tot / el_s, "unit": UNIT, "h2d_bytes_per_step": 4 * d,
            "d2h_bytes_per_step": (local_rows * d * 4 if mode == "materialize" else 0) + 16,
            "bytes_per": "rank and step",
            "steps": steps, "timing": "host wall clock around synchronised steps, max over ranks",
            "api": ("fz_run_host (gens in host memory -> rows streamed through the device output ring into pinned "
                    "host memory), one element per rank" if mode == "materialize" else
                    "Layout/Memo/Plan (gens H2D each step) + all_reduce + fz_plan_result (16 B D2H)")}


def cpu_baseline(W, budget_s: float = 12.0):
    """The oracle as it stands (O1 nested loop + R17 hash, OpenMP over a_1) on this host's cores,
    on a bounded sample of the same workload: the a_1 range is cut into 64 contiguous chunks, visited
    from the fewest rows up (predicted by the oracle's GF counts) until the next chunk would overrun
    the budget at the rate measured so far (C2: the whole workload; C4: its high-a_1 chunks)."""
    from oracle import oracle as O

    g, n = W["gens"], W["n"]
    C = O.C()
    threads = len(os.sched_getaffinity(0))
    top = n // g[0]
    nch = 64
    bounds = [(top + 1) * c // nch for c in range(nch + 1)]
    tail = C.gf_table(n, tuple(g[1:])) if len(g) > 1 else None      # |Z(x; g_2..g_d)|, x <= n

    def est(c):
        if tail is None:
            return 1
        return sum(int(tail[n - a * g[0]]) for a in range(bounds[c], bounds[c + 1]))
    ests = {c: est(c) for c in range(nch)}
    order = sorted(range(nch), key=lambda c: ests[c])
    rows, el, done = 0, 0.0, 0
    t0 = time.perf_counter()
    for c in order:
        lo, hi = bounds[c], bounds[c + 1] - 1
        if el > 0.2 and rows and ests[c] / (rows / el) > budget_s - el:
            break
        if hi >= lo:
            r, _h = C.count_hash(n, g, use_o2=False, threads=threads, a1_range=(lo, hi))
            rows += r
        done += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    full = done == nch
    return {"value": rows / max(el, 1e-9), "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": (f"{done}/{nch} a_1 chunks of Z({n}; {','.join(map(str, g))}), fewest rows first "
                       f"({'complete workload' if full else 'bounded sample'}; {rows} rows), O1 nested loop + "
                       f"R17 hash, {threads} OpenMP threads, {el:.1f} s"),
            "seconds": el}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on this host (rank 0 only), same config/metric/unit."""
    if rank != 0:
        return None
    n_gpus = max(world, args.gpus)
    W = workload(args.config or ("C2" if n_gpus == 1 else "C4"), 0, 1)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(W, budget_s=per_step / 4)
    vals, secs = [], 0.0
    last = None
    for _ in range(args.steps):
        last = cpu_baseline(W, budget_s=per_step)
        vals.append(last["value"])
        secs += last["seconds"]
    v = sorted(vals)[len(vals) // 2]
    last["value"] = v
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3 / max(1, args.steps), "higher_is_better": True,
            "scaling": "strong" if W["mode"] == "count" else "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": f"{W['name']}: Z(n; {','.join(map(str, W['gens']))}) {W['mode']} (CPU oracle sample)",
                       "n": W["n"], "gens": list(W["gens"]), "t": W["t"], "mode": W["mode"]},
            "cpu_baseline": last,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------ f4 study (not part of the default run)
def cpu_baseline_memo(g, t: int, top: int, reps: int = 3) -> float:
    """The paper's CPU memo variant (Alg. LexicographicFactorizationListsUpToElement, PAPER.md:139-153,
    single thread; Table 1's cpu_memo_us column) as the oracle implements it (orc_memo_alg2),
    timed on this host: the CPU side of the f4 CPU-vs-GPU memo crossover.  Microseconds,
    median of `reps`."""
    from oracle import oracle as O

    C, tail = O.C(), tuple(g[len(g) - t:])
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        C.memo_alg2(tail, top)
        ts.append((time.perf_counter() - t0) * 1e6)
    return sorted(ts)[len(ts) // 2]


def f4_study(args):
    """SURVEY §8(f) f4 (PAPER.md:194 both memo variants timed; PAPER.md:301 the best memoDim depends on the
    instance): for Table 1's 31 rows (materialize), C2 (materialize), C3 (hash) and C4 (count), the whole-step
    time (memo build + plan + K5, CUDA events, median of 5) for every memo dimension t the cost model does not
    rule out by 30x, the GPU memo build alone and, for Table 1 rows, the single-thread CPU memo (oracle Alg 2)
    at the paper's t.  One JSON object per line; tools/f4_fit.py fits fz_recommend_t's constants to it."""
    import torch

    from fzinputs import C2, C3_GENS, C3_N, C4, TABLE1_ROWS, table1_gens
    from paper_2407_20474_b200 import fz

    fz.set_memo_cap(64 << 30)

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

    cases = [(f"T1 d={d} n={n}", table1_gens(d), n, "materialize", md) for d, md, n in TABLE1_ROWS]
    cases += [("C2", C2.gens, C2.n, "materialize", C2.t), ("C3", C3_GENS, C3_N, "hash", 3), ("C4", C4.gens, C4.n,
                                                                                              "count", C4.t)]
    for name, g, n, mode, tp in cases:
        d = len(g)
        _, pred = fz.recommend_t(g, n, mode)
        best_pred = min(pred.values()) if pred else None
        rec = {"case": name, "gens": list(g), "n": n, "mode": mode, "t_paper": tp, "pred_s": pred, "step_us": {},
               "memo_us": {}}
        for t in range(1, d):
            if t not in pred or pred[t] > 30 * best_pred:
                continue
            try:
                lay = fz.Layout(g, t, n + 1, entries=mode != "count")
            except fz.FzError:
                continue
            ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
            memo = fz.Memo(layout=lay, workspace=ws)
            pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device="cuda")
            rows = fz.Plan(memo, n, mode, workspace=pws).rows
            out = torch.empty((max(rows, 1), d), dtype=torch.int32, device="cuda") if mode == "materialize" else None

            def step():
                m = fz.Memo(layout=lay, workspace=ws)
                fz.Plan(m, n, mode, workspace=pws).launch(out)
            reps = 3 if pred[t] > 0.05 else 5
            rec["step_us"][t] = timed(step, reps=reps, warm=1 if pred[t] > 0.05 else 2)
            rec["memo_us"][t] = timed(lambda: fz.Memo(layout=lay, workspace=ws), reps=5)
            del out, ws
        if name.startswith("T1"):
            rec["cpu_memo_us"] = cpu_baseline_memo(g, tp, n + 1)
        print(json.dumps(rec), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(args) -> int:
    """`python bench.py --gpus N` outside torchrun: run the N ranks under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default=None, choices=["C2", "C2batch", "C4", "C4t2"],
                    help="headline workload (default: C2 at N = 1, C4 at N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-count", action="store_true", help="skip the extra legs")
    ap.add_argument("--no-hash", action="store_true")
    ap.add_argument("--study", default=None, choices=["f4"], help="run a study instead of the bench line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)

    if args.study == "f4":
        f4_study(args)
        return
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))

    import torch
    import torch.distributed as dist

    ngpu = max(1, torch.cuda.device_count())
    backend = "none"
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # one process per GPU over NCCL; with fewer GPUs than ranks (or FZ_BENCH_BACKEND=gloo) the ranks
        # share GPUs over gloo (NCCL refuses two ranks on one device) and the line says so
        backend = os.environ.get("FZ_BENCH_BACKEND", "nccl" if ngpu >= world else "gloo")
        local_rank = local_rank % ngpu
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            ver = ".".join(map(str, torch.cuda.nccl.version()))
            backend = f"nccl {ver} ({world} ranks on {world} GPUs)"
        else:
            dist.init_process_group("gloo")
            backend = f"gloo ({world} ranks sharing {ngpu} GPU{'s' if ngpu > 1 else ''})"
        if rank == 0:
            print(f"[bench] communicator: {backend}", file=sys.stderr, flush=True)
    res, W, _ = run_native(args, rank, world, local_rank, backend)
    if not args.no_e2e:
        res["e2e"] = run_e2e(args, W, rank, world, local_rank)
    if not args.no_count:
        res["legs"] = native_legs(args, rank, world, local_rank, W["name"])
    if rank == 0:
        if world == 1 and not args.no_cpu:
            res["cpu_baseline"] = cpu_baseline(W)
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
