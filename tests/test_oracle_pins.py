"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/) is checked against things other than itself: the paper's
printed Table 1 counts, SPEC.md's worked examples, brute
force on tiny inputs, the independent generating-function count, the d = 2
closed form, known-answer hash vectors from SURVEY App. A, and structural
invariants (strict descending order, phi = n, recurrence identities).  Each is
chosen so that a plausible slip (dropped term, wrong index, reversed order,
transposed operand) fails at least one test.
"""
import math
import os

import numpy as np
import pytest

from conftest import parse_gens, read_golden_csv
from fzinputs import random_instance, random_instance_mid, table1_gens
from oracle import oracle as O

GOLDEN_SPEC = __import__("os").path.join(__import__("conftest").GOLDEN, "spec_examples.txt")


def _rows(s, d):
    if s == "-":
        return []
    return [tuple(int(x) for x in r.split(",")) for r in s.split(";")]


def _spec_cases(kind):
    out = []
    for line in open(GOLDEN_SPEC):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f = [x.strip() for x in line.split("|")]
        if f[0] == kind:
            out.append(f[1:])
    return out


# ------------------------------------------------------------- SPEC examples
@pytest.mark.parametrize("case", _spec_cases("list"), ids=lambda c: f"Z({c[1]};{c[0]})")
def test_spec_lists(case, corc):
    g = tuple(int(x) for x in case[0].split(","))
    n = int(case[1])
    want = _rows(case[2], len(g))
    assert O.brute_force(n, g) == want
    assert O.enum_py(n, g) == want
    assert O.alg2_lists(n, g)[n] == want
    for o2 in (False, True):
        rows, cnt, _ = corc.enumerate(n, g, use_o2=o2)
        assert cnt == len(want)
        assert [tuple(int(v) for v in r) for r in rows] == want
    assert O.gf_count_py(n, g) == len(want)


@pytest.mark.parametrize("case", _spec_cases("memo"), ids=lambda c: f"memo({c[0]};{c[1]})")
def test_spec_memo(case, corc):
    h = tuple(int(x) for x in case[0].split(","))
    top = int(case[1])
    want = [int(x) for x in case[2].split(",")]
    F = O.alg2_lists(top - 1, h, top=top)
    assert [x for x in range(top) if F[x]] == want
    assert max(len(F[x]) for x in range(top)) == 1          # maxSetCardinality = 1
    rows, off = corc.memo_alg2(h, top)
    assert [x for x in range(top) if off[x + 1] > off[x]] == want
    flat = [r for x in range(top) for r in F[x]]
    assert [tuple(int(v) for v in r) for r in rows] == flat


@pytest.mark.parametrize("case", _spec_cases("trace"), ids=lambda c: f"trace({c[1]};{c[0]};t={c[2]})")
def test_spec_traces(case):
    """SPEC.md:303-313 hand traces of nextCandidate / nextCandidateDynamic."""
    g = tuple(int(x) for x in case[0].split(","))
    n, md = int(case[1]), int(case[2])
    want = []
    for item in case[3].split(";"):
        a, v = item.split(":")
        want.append((tuple(int(x) for x in a.split(",")), bool(int(v))))
    st = O.set_initial_candidate(n, g)
    got = []
    if md == 0:
        while True:
            O.next_candidate(st, n, g)
            if st["endOfStream"] and not st["wasValid"] and (not got or tuple(st["a"]) == got[-1][0]):
                break
            got.append((tuple(st["a"]), st["wasValid"]))
            if st["endOfStream"]:
                break
    else:
        memo = O.alg2_lists(n, g[len(g) - md:])
        while not st["endOfStream"]:
            O.next_candidate_dynamic(st, n, g, memo, md, n + 1)
            got.append((tuple(st["a"]), st["wasValid"]))
    assert got == want
    assert O.alg5_run(n, g, max(md, 1)) == O.brute_force(n, g)


def test_spec_memo_trace_outputs():
    """the only memo hit with output is a=(1,0,0), p=18 -> (1,2,0)."""
    g, n = (6, 9, 20), 24
    st = O.set_initial_candidate(n, g)
    assert st["a"] == [4, 0, 0] and st["wasValid"]
    memo = O.alg2_lists(n, (9, 20))
    outs = []
    while not st["endOfStream"]:
        outs.append(O.next_candidate_dynamic(st, n, g, memo, 2, n + 1))
    assert outs == [[], [], [(1, 2, 0)], []]


def test_initial_candidate_examples():
    """SPEC.md:293-295."""
    assert O.set_initial_candidate(6, (2, 3))["a"] == [3, 0]
    s = O.set_initial_candidate(7, (2, 3))
    assert s["a"] == [4, 0] and not s["wasValid"]
    s = O.set_initial_candidate(0, (2, 3))
    assert s["a"] == [0, 0] and s["wasValid"]


# ------------------------------------------------------------------ Table 1
TABLE1 = read_golden_csv("table1.csv")


@pytest.mark.parametrize("row", TABLE1, ids=lambda r: f"L{r['paper_line']}-d{r['dim']}-n{r['element']}")
def test_table1_counts(row, corc):
    """num_results column of Table 1 against the GF count (u128)
    and the O2 nested loop.  Line 318 is the erratum R14: the paper prints 779252,
    both independent oracles give 779257."""
    d, n = int(row["dim"]), int(row["element"])
    g = table1_gens(d)
    printed = int(row["num_results"])
    gf = corc.gf_count(n, g)
    if row["paper_line"] == "318":
        assert printed == 779252 and gf == 779257
    else:
        assert gf == printed
    if gf <= 3_000_000:
        cnt, _ = corc.count_hash(n, g, use_o2=True, threads=0)
        assert cnt == gf
    if gf <= 300_000:
        cnt1, _ = corc.count_hash(n, g, use_o2=False, threads=0)
        assert cnt1 == gf


@pytest.mark.parametrize("d,md,n", [(4, 2, 5000), (5, 3, 1000), (9, 5, 500), (9, 4, 500), (6, 3, 1000)])
def test_table1_alg5_small(d, md, n, corc):
    """The paper's own Alg 5 (single stream, Python) reproduces Table 1 rows and the O1 list."""
    g = table1_gens(d)
    out = O.alg5_run(n, g, md)
    rows, cnt, _ = corc.enumerate(n, g)
    assert len(out) == cnt
    assert out == [tuple(int(v) for v in r) for r in rows]


# ------------------------------------------------------ random O0 equivalence
def _bf_feasible(n, g, cap=60_000):
    return math.prod(n // x + 1 for x in g) <= cap


@pytest.mark.parametrize("seed", range(200))
def test_random_equivalence(seed, corc):
    """>= 200 random instances (d 2..5, g_i <= 25, n <= 120).  O0 (brute
    force), O1 (Python and C), O2, Alg 2, Alg 3, Alg 5 (every memo_dim, three tops)
    and the GF count must agree; Alg 1 as sets."""
    g, n, _ = random_instance(seed)
    ref = O.enum_py(n, g)
    if _bf_feasible(n, g):
        assert O.brute_force(n, g) == ref
    assert len(ref) == O.gf_count_py(n, g) == corc.gf_count(n, g)
    for o2 in (False, True):
        rows, cnt, h = corc.enumerate(n, g, use_o2=o2)
        assert cnt == len(ref)
        assert [tuple(int(v) for v in r) for r in rows] == ref
        assert h == O.hash_list(ref)
    assert O.alg2_lists(n, g)[n] == ref
    Z3, _ = O.alg3_cardinalities(n, g)
    assert Z3[n] == ref
    assert O.alg1_sets(n, g)[n] == set(ref)
    for md in range(1, len(g)):
        for top in sorted({1, n // 2 + 1, n + 1}):
            assert O.alg5_run(n, g, md, top=top) == ref
    # invariants: strictly descending, phi = n
    assert all(ref[i] > ref[i + 1] for i in range(len(ref) - 1))
    assert all(O.phi(a, g) == n for a in ref)


@pytest.mark.parametrize("seed", range(12))
def test_mid_instances_o1_o2_gf(seed, corc):
    """Mid-size instances (Table-1-shaped generators): O1 == O2 lists, count == GF,
    parallel count_hash == serial hash, shard-additivity of the hash."""
    g, n, _ = random_instance_mid(seed)
    rows1, c1, h1 = corc.enumerate(n, g, use_o2=False)
    rows2, c2, h2 = corc.enumerate(n, g, use_o2=True)
    assert c1 == c2 == corc.gf_count(n, g)
    assert np.array_equal(rows1, rows2) and h1 == h2
    if c1:
        assert np.all(rows1.astype(np.int64) @ np.array(g, dtype=np.int64) == n)
        r = rows1.astype(np.int64)
        # strictly descending lex: first differing coordinate decreases
        diff = r[:-1] - r[1:]
        first = np.argmax(diff != 0, axis=1)
        assert np.all(diff[np.arange(len(diff)), first] > 0)
    for th in (1, 4):
        assert corc.count_hash(n, g, use_o2=True, threads=th) == (c1, h1)
        assert corc.count_hash(n, g, use_o2=False, threads=th) == (c1, h1)
    k = c1 // 3
    assert (corc.hash_rows(rows1[:k]) + corc.hash_rows(rows1[k:], row_base=k)) % (1 << 64) == h1


def test_count_hash_a1_ranges_partition(corc):
    """count_hash over disjoint a_1 ranges sums to the whole (used by cpu_baseline samples)."""
    g, n = (13, 37, 38, 40), 5000
    full = corc.count_hash(n, g)
    top = n // 13
    parts = [corc.count_hash(n, g, a1_range=(lo, min(lo + 49, top))) for lo in range(0, top + 1, 50)]
    assert sum(p[0] for p in parts) == full[0]
    assert sum(p[1] for p in parts) % (1 << 64) == full[1]


# --------------------------------------------------------- d = 2 closed form
@pytest.mark.parametrize("seed", range(40))
def test_d2_closed_form(seed, corc):
    import random

    r = random.Random(seed)
    for _ in range(75):
        a, b = r.randint(1, 60), r.randint(1, 60)
        n = r.randint(0, 3000)
        want = O.d2_count(n, a, b)
        assert O.gf_count_py(n, (a, b)) == want
        assert len(O.enum_py(n, (a, b))) == want


def test_gf_closed_forms():
    """Single generator: [g | n]; all-ones d gens: C(n+d-1, d-1)."""
    for gi in (1, 2, 7):
        for n in range(30):
            assert O.gf_count_py(n, (gi,)) == (1 if n % gi == 0 else 0)
    for d in (2, 3, 5):
        for n in (0, 1, 9, 40):
            assert O.gf_count_py(n, (1,) * d) == math.comb(n + d - 1, d - 1)


# ------------------------------------------------------------------ hashing
HASH_KATS = read_golden_csv("hash_kats.csv")


@pytest.mark.parametrize("kat", [k for k in HASH_KATS if k["tier"] == "small"],
                         ids=lambda k: f"{k['gens']}-{k['n']}")
def test_hash_kats(kat, corc):
    g, n = parse_gens(kat["gens"]), int(kat["n"])
    want = (int(kat["count"]), int(kat["H"], 16))
    assert corc.count_hash(n, g, use_o2=True) == want
    if want[0] <= 3_000_000:
        assert corc.count_hash(n, g, use_o2=False) == want
    if want[0] <= 600:
        rows = O.enum_py(n, g)
        assert (len(rows), O.hash_list(rows)) == want


@pytest.mark.slow
@pytest.mark.parametrize("kat", [k for k in HASH_KATS if k["tier"] == "mid"],
                         ids=lambda k: f"{k['gens']}-{k['n']}")
def test_hash_kats_mid(kat, corc):
    g, n = parse_gens(kat["gens"]), int(kat["n"])
    assert corc.count_hash(n, g, use_o2=True) == (int(kat["count"]), int(kat["H"], 16))


@pytest.mark.slow
@pytest.mark.parametrize("kat", [k for k in HASH_KATS if k["tier"] == "big"],
                         ids=lambda k: f"{k['gens']}-{k['n']}")
def test_hash_kats_big(kat, corc):
    """The big-tier KATs (C3: Z(17350; 23..43), 1.0e10 rows; the C4 shape Z(10000; 97..104), 2.5e8 rows)
    reproduced by oracle/ itself (O2 + R17, OpenMP over a_1): closes the chain from SURVEY App. A's scratch
    values to the constants the GPU tests assert (test_c3_count_hash, test_c4_shape_hash).  ~1-2 min on 8 cores."""
    g, n = parse_gens(kat["gens"]), int(kat["n"])
    assert corc.count_hash(n, g, use_o2=True, threads=len(os.sched_getaffinity(0))) == \
        (int(kat["count"]), int(kat["H"], 16))


def test_hash_properties():
    """Order sensitivity (reversing the list changes H) and row_base additivity."""
    rows = O.enum_py(200, (6, 9, 20))
    h = O.hash_list(rows)
    assert O.hash_list(rows[::-1]) != h
    # SURVEY App. A KAT: Z(24;6,9,20) in reversed (ascending) order -> 0xf021eecaebeb2124
    z = O.enum_py(24, (6, 9, 20))
    assert O.hash_list(z) == 0xBFECD72A6F34D2FA and O.hash_list(z[::-1]) == 0xF021EECAEBEB2124
    k = len(rows) // 2
    assert (O.hash_list(rows[:k]) + O.hash_list(rows[k:], row_base=k)) % (1 << 64) == h
    assert O.hash_list([]) == 0


def test_c1_aggregate():
    """sum_{m<=1000} |Z(m;6,9,20)| = 162781 and sum of H(Z(m)) = 0x54c291a6f228ca38."""
    C = O.C()
    tot, hs = 0, 0
    for m in range(1001):
        c, h = C.count_hash(m, (6, 9, 20), threads=1)
        tot += c
        hs = (hs + h) % (1 << 64)
    assert tot == 162781 and hs == 0x54C291A6F228CA38


# -------------------------------------------------------------------- memo
MEMO_KATS = read_golden_csv("memo_kats.csv")


@pytest.mark.parametrize("kat", [k for k in MEMO_KATS if k["tier"] == "small"],
                         ids=lambda k: f"{k['tail']}-{k['top']}")
def test_memo_kats(kat, corc):
    """Alg 2 over the tail generators (the memo) against SURVEY App. A."""
    h, top = parse_gens(kat["tail"]), int(kat["top"])
    rows, off = corc.memo_alg2(h, top)
    assert int(off[top]) == int(kat["entries"])
    assert corc.hash_rows(rows) == int(kat["H"], 16)
    # per-x block == Z(x; tail) from the GF count and O1 on a sample of x
    tbl = corc.gf_table(top - 1, h)
    assert np.array_equal(np.diff(off.astype(np.int64)), tbl.astype(np.int64))
    for x in list(range(0, min(top, 60))) + list(range(top - 5, top)):
        r1, _, _ = corc.enumerate(x, h)
        assert np.array_equal(rows[int(off[x]):int(off[x + 1])], r1)


@pytest.mark.parametrize("seed", range(10))
def test_cardinality_identity(seed):
    """SPEC.md:461 / PAPER.md:163-166: C[m][i] = sum_{j>=i} C[m-g_i][j] and the slices
    tile Z(m) in order i = 1..d with slice i = {a : a_j = 0 (j<i), a_i > 0}."""
    import random

    r = random.Random(seed)
    d = r.randint(2, 4)
    g = tuple(r.randint(2, 12) for _ in range(d))
    Z, C = O.alg3_cardinalities(300, g)
    for m in range(1, 301):
        assert sum(C[m]) == len(Z[m])
        pos = 0
        for i in range(d):
            if m >= g[i]:
                assert C[m][i] == sum(C[m - g[i]][i:])
            sl = Z[m][pos:pos + C[m][i]]
            assert all(all(a[j] == 0 for j in range(i)) and a[i] > 0 for a in sl)
            pos += C[m][i]
        assert Z[m] == O.enum_py(m, g)
