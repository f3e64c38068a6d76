"""CPU checks of bench.py's host-side bookkeeping (no GPU): the COUNT roofline's unit count, the
workload table against BASELINE.json's configs, and the cpu_baseline / reference-arm record."""
import itertools
import json
import os

import bench
from conftest import ROOT
from fzinputs import C2, C4


def _prefixes_brute(g, n, L):
    """Leading prefixes (a_1..a_L) with sum a_i g_i <= n, by enumeration."""
    gl = g[:L]
    ranges = [range(n // x + 1) for x in gl]
    return sum(1 for a in itertools.product(*ranges) if sum(ai * gi for ai, gi in zip(a, gl)) <= n)


def test_leading_prefixes_matches_enumeration():
    for g, n, L in [((3, 5, 7, 11), 40, 2), ((2, 3), 17, 1), ((4, 6, 9, 10, 15), 30, 3), ((7,), 50, 1),
                    ((6, 9, 20), 100, 2)]:
        assert bench.leading_prefixes(g, n, L) == _prefixes_brute(g, n, L), (g, n, L)


def test_c4_prefix_count_is_survey_figure():
    # C4 t = 3 walks 9.26e10 leading prefixes
    u = bench.leading_prefixes(C4.gens, C4.n, len(C4.gens) - C4.t)
    assert 9.25e10 < u < 9.27e10


def test_workloads_follow_baseline_configs(corc):
    cfgs = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert "11,13,17,19" in cfgs[1].replace(" ", "") and "1e8" in cfgs[1]
    # configs[1]'s "single large n yielding ~1e8 factorizations": the first n with |Z(n)| >= 1e8 (GF count)
    assert corc.gf_count(C2.n, C2.gens) >= 10**8 > corc.gf_count(C2.n - 1, C2.gens)
    w = bench.workload("C2", 0, 1)
    assert (w["gens"], w["n"], w["mode"], w["scaling"]) == (C2.gens, 30232, "materialize", "weak")
    w = bench.workload("C2", 3, 8)                                                # one element row-sharded
    assert (w["n"], w["shard"], w["nshards"], w["scaling"]) == (30232, 3, 8, "strong")
    w = bench.workload("C2batch", 3, 8)
    assert w["n"] == 30232 - 3 and w["nshards"] == 1 and w["scaling"] == "weak"   # one element per rank
    w = bench.workload("C4", 5, 8)
    assert (w["shard"], w["nshards"], w["mode"], w["scaling"]) == (5, 8, "count", "strong")
    # configs[3] ("d=8 generators near 100, large n count-only, sharded ... over 2/4/8"): the N > 1 headline
    assert "d=8" in cfgs[3] and "count" in cfgs[3] and len(C4.gens) == 8 and all(90 < x < 110 for x in C4.gens)


def test_cpu_baseline_record():
    rec = bench.cpu_baseline(bench.workload("C2", 0, 1), budget_s=0.3)
    assert rec["kind"] == "oracle" and rec["unit"] == bench.UNIT
    assert rec["cores"] >= 1 and rec["value"] > 0 and rec["seconds"] > 0
    assert "a_1 chunks" in rec["sample"]


def test_spawn_command(monkeypatch):
    """`python bench.py --gpus N` outside torchrun re-runs itself under torch.distributed.run with N ranks
    on 127.0.0.1 (the command is built, not run)."""
    import sys

    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])

    class A:
        gpus = 4
    bench.spawn(A)
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-4:] == ["--gpus", "4", "--steps", "3"]
