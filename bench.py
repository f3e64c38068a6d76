"""bench.py -- factorizations/sec of the whole hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--config C2|C4]

A step is one pass of the whole hot path over one element:
memo build on the GPU (count pass K1 + copy-increment recurrence K3), device-side shard
plan K4, enumeration K5 (materialize for C2, count for C4) and, for N > 1 with one problem
cut into shards (C4), the NCCL all-reduce of the {rows, hash} accumulators (A10); the weak C2
batch has no data-path collective.  The A1 host layout (validation + sizing,
like an FFT plan) is made once per configuration, outside the timed region.

N = 1 runs BASELINE.json configs[1] (C2: Z(30232; 11,13,17,19), ~1e8 rows materialized).
For N > 1 (torchrun, one process per GPU) C2 is a batch of N independent elements, one per
GPU (n_r = 30232 - r): per-GPU work fixed -> "scaling": "weak"; --config C4 instead splits
ONE count problem (Z(40000; 97..104), 3.36e12 rows) across the ranks -> "strong".

`--impl reference` times the CPU oracle (oracle/, the plain nested-loop definition) on this
host's cores on a bounded sample of the same workload (there is no reference program to
install: the reference is a paper).
"""
from __future__ import annotations

import argparse
import json
import os
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


def workload(cfg: str, rank: int, world: int):
    from fzinputs import C2, C4

    if cfg == "C2":
        return dict(name="C2", gens=C2.gens, n=C2.n - rank, t=C2.t, mode="materialize", shard=0, nshards=1,
                    scaling="weak")
    if cfg == "C4":
        return dict(name="C4", gens=C4.gens, n=C4.n, t=C4.t, mode="count", shard=rank, nshards=world,
                    scaling="strong")
    raise SystemExit(f"unknown --config {cfg}")


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


# ------------------------------------------------------------------ native arm
def run_native(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2407_20474_b200 import fz

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    W = workload(args.config, rank, world)
    g, n, t, mode = W["gens"], W["n"], W["t"], W["mode"]
    entries = mode != "count"
    lay = fz.Layout(g, t, n + 1, entries=entries)                  # A1 (host, once)
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device=dev)
    memo = fz.Memo(layout=lay, workspace=ws)
    pws = torch.empty(fz.plan_workspace_bytes(memo), dtype=torch.uint8, device=dev)
    plan = fz.Plan(memo, n, mode, W["shard"], W["nshards"], workspace=pws)
    rows_expect = plan.rows
    out = torch.empty((max(rows_expect, 1), len(g)), dtype=torch.int32, device=dev) if mode == "materialize" else None
    stream = torch.cuda.current_stream()

    def step(ev_k5=None):
        m = fz.Memo(layout=lay, workspace=ws)                          # K1 + K3
        p = fz.Plan(m, n, mode, W["shard"], W["nshards"], workspace=pws)   # K4
        if ev_k5 is not None:
            ev_k5[0].record(stream)
        p.launch(out)                                                   # K5
        if ev_k5 is not None:
            ev_k5[1].record(stream)
        if world > 1 and W["scaling"] == "strong":
            # A10: {rows, hash} of the shards of ONE problem (the weak C2 batch has independent
            # elements per rank: no data-path collective)
            dist.all_reduce(p.result_tensor(), op=dist.ReduceOp.SUM)
        return m, p

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    m0, p0 = step()
    torch.cuda.synchronize()
    r_step, h_step = p0.result()
    if world == 1 or W["scaling"] == "weak":
        assert r_step == rows_expect, (r_step, rows_expect)
    if world > 1 and W["scaling"] == "weak":   # rows of the whole batch, once, outside the timed region
        rt = torch.tensor([r_step], dtype=torch.float64, device=dev)
        dist.all_reduce(rt, op=dist.ReduceOp.SUM)
        r_step = int(rt.item())

    k5_events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(args.steps)]
    launches0 = fz.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record(stream)
        keep = []
        for k in range(args.steps):
            keep.append(step(k5_events[k]))
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = fz.launch_count() - launches0
    ms_total = e0.elapsed_time(e1)
    k5_ms = sum(a.elapsed_time(b) for a, b in k5_events) / args.steps
    tt = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_total = float(tt.item())
    # r_step: every rank's rows of the step (N > 1: the all-reduced shard accumulators, or the batch sum)
    rows_per_step = float(r_step)
    value = rows_per_step * args.steps / (ms_total / 1e3)
    r_local = rows_expect

    # roofline of the dominant kernel (K5): algorithmic bytes per launch / its event time
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    if mode == "materialize":
        alg_bytes = r_local * len(g) * 4
        peak = peaks.get("hbm_gbs")
        roof = {"kernel": f"k5_walk<{len(g)},{t},materialize>", "bound": "hbm",
                "achieved": alg_bytes / (k5_ms / 1e3) / 1e9, "peak": peak if peak else 6650.0,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if peak else "fallback (B200_PROFILING.md)",
                "unit": "GB/s", "algorithmic_bytes_per_launch": alg_bytes}
        roof["frac"] = roof["achieved"] / roof["peak"]
    else:
        # COUNT: one card lookup per leading prefix, 2 B each from the shared-memory copy
        # of the card table; bound: the shared-memory crossbar, 128 B/clk/SM (B300_MICROARCH.md, LDS/STS)
        # -> SMs x 128 / 2 lookups per clock at the max SM clock
        U = leading_prefixes(g, n, len(g) - t)
        # N > 1: the COUNT shards are cost-balanced, not unit-balanced; U / N is their mean
        units = U // W["nshards"]
        props = torch.cuda.get_device_properties(dev)
        clk = sampler.summary().get("sm_max_mhz") or 1965
        peak = props.multi_processor_count * 128 / 2 * clk * 1e6
        roof = {"kernel": f"k5_walk<{len(g)},{t},count>", "bound": "alu", "achieved": units / (k5_ms / 1e3),
                "unit": "card lookups/s (leading prefixes)", "peak": peak,
                "peak_source": "derived: SMs x 128 B/clk shared-memory crossbar / 2 B per u16 card x max SM clock",
                "algorithmic_units_per_launch": units, "frac": units / (k5_ms / 1e3) / peak}
        if W["nshards"] > 1:
            roof["units_note"] = "mean units per shard (cost-balanced COUNT cut)"
    roof["traffic"] = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "k5_traffic.json")))
        key = f"{W['name']}"
        if key in prof:
            roof["traffic"] = prof[key]["dram_bytes_per_launch"]
    except Exception:
        pass
    roof["k5_ms"] = k5_ms

    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": W["scaling"], "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (fixed generator tuples; no datasets)",
        "config": {"workload": f"{W['name']}: Z(n; {','.join(map(str, g))}) {mode}, memo t={t}, top=n+1",
                   "n": n, "gens": list(g), "t": t, "mode": mode, "rows_per_rank_step": r_local,
                   "fill_mode": lay.info["fill_mode"],
                   "l2": ("each step writes its 1.6 GB output (> 126 MB L2), flushing L2 between steps"
                          if mode == "materialize" else "count mode: tables L2-resident by design"),
                   "parallelism": f"{'batch' if W['scaling'] == 'weak' else 'shard'}{world}"},
        "gpu_launches": launches,
        "roofline": roof,
        "clocks": sampler.summary(),
    }
    if world > 1:
        res["config"]["collective"] = ("NCCL all_reduce(SUM) of the {rows, hash} shard accumulators each step"
                                       if W["scaling"] == "strong" else
                                       "none in the data path (independent elements per rank)")
    return res, (g, n, t, mode)


def count_mode_extra(local_rank):
    """Count mode (the metric's second half) on this GPU: C2's element and C4 (t=3), whole step
    (count tables + plan + the COUNT walk over every leading prefix), CUDA-event timed."""
    import torch

    from fzinputs import C2, C4
    from paper_2407_20474_b200 import fz

    res = {}
    for name, g, n, t, steps in (("C2", C2.gens, C2.n, C2.t, 50), ("C4", C4.gens, C4.n, C4.t, 5)):
        lay = fz.Layout(g, t, n + 1, entries=False)
        ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
        pws = torch.empty(256, dtype=torch.uint8, device="cuda")

        def step():
            m = fz.Memo(layout=lay, workspace=ws)
            p = fz.Plan(m, n, "count", workspace=pws)
            p.launch()
            return m, p
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        keep = [step() for _ in range(steps)]
        e1.record()
        torch.cuda.synchronize()
        rows, _ = keep[-1][1].result()
        ms = e0.elapsed_time(e1) / steps
        res[name] = {"value": rows / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "rows": rows, "t": t,
                     "workload": f"Z({n}; {','.join(map(str, g))}) count, t={t}"}
    return res


def hash_mode_extra(local_rank):
    """Hash mode on BASELINE.json configs[2] (C3: Z(17350; 23,29,31,37,41,43), 1.0e10 rows, t = 3 — the
    fastest memo dimension): whole step (memo build + plan + the HASH walk), CUDA-event timed; the
    (count, H) pair is compared with the known answer in tests/golden/hash_kats.csv."""
    import torch

    from fzinputs import C3_GENS, C3_N
    from paper_2407_20474_b200 import fz

    g, n, t, steps = C3_GENS, C3_N, 3, 3
    kat = None
    for line in open(os.path.join(ROOT, "tests", "golden", "hash_kats.csv")):
        f = line.strip().split(",")
        if len(f) >= 4 and f[0] == ";".join(map(str, g)) and f[1] == str(n):
            kat = (int(f[2]), int(f[3], 16))
    lay = fz.Layout(g, t, n + 1, entries=True)
    ws = torch.empty(lay.workspace_bytes, dtype=torch.uint8, device="cuda")
    pws = None

    def step():
        nonlocal pws
        m = fz.Memo(layout=lay, workspace=ws)
        if pws is None:
            pws = torch.empty(fz.plan_workspace_bytes(m), dtype=torch.uint8, device="cuda")
        p = fz.Plan(m, n, "hash", workspace=pws)
        p.launch()
        return m, p
    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    keep = [step() for _ in range(steps)]
    e1.record()
    torch.cuda.synchronize()
    rows, h = keep[-1][1].result()
    ms = e0.elapsed_time(e1) / steps
    return {"C3": {"value": rows / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "rows": rows, "t": t,
                   "hash": f"{h:#018x}", "kat_match": kat == (rows, h),
                   "workload": f"Z({n}; {','.join(map(str, g))}) hash, t={t}"}}


def run_e2e(args, spec, W, rank, world, local_rank):
    """Same metric end to end through the public API from HOST buffers, on every rank; the timed region
    (barrier-bracketed, max over ranks) holds each step's H2D of the generator tuple and D2H of the result.
    MATERIALIZE (weak, one element per rank): fz_run_host, rows streamed into pinned host memory.
    COUNT (strong, one problem cut into shards): this rank's shard through Layout/Memo/Plan with the
    NCCL all_reduce of {rows, hash}, then the 16-byte D2H read of the global result."""
    import torch
    import torch.distributed as dist

    from paper_2407_20474_b200 import fz

    g, n, t, mode = spec
    d = len(g)
    dev = torch.device("cuda", local_rank)
    steps = max(1, min(args.steps, 3))
    host = None
    if mode == "materialize":
        ws = torch.empty(fz.run_workspace_bytes(g, t, n, mode), dtype=torch.uint8, device=dev)
        lay = fz.Layout(g, t, n + 1, entries=True)
        rows = fz.Plan(fz.Memo(layout=lay), n, mode).rows
        host = torch.empty((rows, d), dtype=torch.int32).pin_memory()

        def one():
            return fz.run_host(g, t, n, mode, host, workspace=ws)[0]
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
            if world > 1:
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
        tot = float(sm[1]) if W["scaling"] == "weak" else float(el[1])   # strong: all_reduced already
    else:
        el_s = float(el[0])
    local_rows = int(el[1].item()) // steps
    return {"value": tot / el_s, "unit": UNIT, "h2d_bytes_per_step": 4 * d,
            "d2h_bytes_per_step": (local_rows * d * 4 if mode == "materialize" else 0) + 16,
            "bytes_per": "rank and step",
            "steps": steps, "timing": "host wall clock around synchronised steps, max over ranks",
            "api": ("fz_run_host (gens in host memory -> rows in pinned host memory), one element per rank"
                    if mode == "materialize" else
                    "Layout/Memo/Plan (gens H2D each step) + all_reduce + fz_plan_result (16 B D2H)")}


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


def cpu_baseline(spec, budget_s: float = 12.0):
    """The oracle as it stands (O1 nested loop + R17 hash, OpenMP over a_1) on this host's cores,
    on a bounded sample of the same workload: the a_1 range is cut into 64 contiguous chunks, visited
    from the fewest rows up (predicted by the oracle's GF counts) until the next chunk would overrun
    the budget at the rate measured so far (C2: the whole workload; C4: its high-a_1 chunks)."""
    from oracle import oracle as O

    g, n, t, mode = spec
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
    W = workload(args.config, 0, 1)
    spec = (W["gens"], W["n"], W["t"], W["mode"])
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(spec, budget_s=per_step / 4)
    vals, secs = [], 0.0
    last = None
    for _ in range(args.steps):
        last = cpu_baseline(spec, budget_s=per_step)
        vals.append(last["value"])
        secs += last["seconds"]
    v = sorted(vals)[len(vals) // 2]
    last["value"] = v
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3 / max(1, args.steps), "higher_is_better": True,
            "scaling": W["scaling"], "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"{W['name']}: Z(n; {','.join(map(str, W['gens']))}) {W['mode']} (CPU oracle sample)",
                       "n": W["n"], "gens": list(W["gens"]), "mode": W["mode"]},
            "cpu_baseline": last,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C4"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-count", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    import torch
    import torch.distributed as dist

    # one process per GPU; FZ_BENCH_BACKEND=gloo lets several ranks share one GPU (CI / single-GPU checks)
    local_rank = local_rank % max(1, torch.cuda.device_count())
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("FZ_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    res, spec = run_native(args, rank, world, local_rank)
    if not args.no_e2e:
        res["e2e"] = run_e2e(args, spec, workload(args.config, rank, world), rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            res["cpu_baseline"] = cpu_baseline(spec)
        if world == 1 and args.config == "C2" and not args.no_count:
            res["count_mode"] = count_mode_extra(local_rank)
            res["hash_mode"] = hash_mode_extra(local_rank)
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
