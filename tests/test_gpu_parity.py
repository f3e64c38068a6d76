"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Integer work, so the bar is bit-exact everywhere: the ordered list (MATERIALIZE), the count
(COUNT) and the 64-bit order-sensitive hash (HASH).  Inputs come from fzinputs (seeded or the
fixed BASELINE configs); every expected value comes from oracle/ or from a cited golden file.
"""
import numpy as np
import pytest
import torch

from conftest import parse_gens, read_golden_csv
from fzinputs import (C1_GENS, C1_MAX_N, C1_T, C2, C3_GENS, C3_N, C4, TABLE1_ROWS, random_instance,
                      random_instance_mid, table1_gens)
from oracle import oracle as O

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2407_20474_b200 import fz


def _np(t):
    return t.cpu().numpy().view(np.uint32)


def _check_materialize(memo, n, corc, g, shards=(1,)):
    want, cnt, h = corc.enumerate(n, g, use_o2=True)
    for ns in shards:
        parts, hs, tot = [], 0, 0
        for s in range(ns):
            out, rows, _ = fz.enumerate(memo, n, "materialize", shard=s, nshards=ns)
            parts.append(_np(out)[:rows])
            tot += rows
            _, hr, hh = fz.enumerate(memo, n, "hash", shard=s, nshards=ns)
            hs = (hs + hh) % (1 << 64)
        got = np.concatenate(parts) if parts else np.zeros((0, len(g)), np.uint32)
        assert tot == cnt, (g, n, ns)
        assert np.array_equal(got.reshape(-1, len(g)), want.reshape(-1, len(g))), (g, n, ns)
        assert hs == h, (g, n, ns)
        crow = 0
        for s in range(ns):
            _, cr, _ = fz.enumerate(memo, n, "count", shard=s, nshards=ns)
            crow += cr
        assert crow == cnt


# ----------------------------------------------------------------- memo (K1-K3)
MEMO_CASES = [((9, 20), 25), ((9, 20), 1001), ((17, 19), 30233), ((41, 43), 17351), ((38, 40), 15001),
              ((38, 40, 41, 42), 3001), ((3, 5, 8), 500), ((1, 1, 2), 200), ((7,), 300), ((4, 6, 10, 4), 400)]


@pytest.mark.parametrize("fill", [0, 1, 2, 3, 4, 5], ids=lambda m: f"fill{m}")
@pytest.mark.parametrize("tail,top", MEMO_CASES, ids=lambda x: str(x))
def test_memo_rows_vs_alg2(tail, top, fill, corc):
    """K1-K3 memo == Alg 2 over the tail generators, row by row, for every
    copy-increment schedule (0 automatic, 1 ring, 2 L2, 3 grid, 4 dimension passes, 5 dimension
    passes in scan form)."""
    g = (5,) + tuple(tail)          # a leading generator, the memo is over the last t = len(tail)
    t = len(tail)
    fz.set_fill_mode(fill)
    try:
        memo = fz.memo_build(g, t, top)
    finally:
        fz.set_fill_mode(0)
    rows, off, S = memo.views()
    want_rows, want_off = corc.memo_alg2(tail, top)
    assert np.array_equal(off.cpu().numpy().astype(np.uint64), want_off)
    assert memo.info["entries"] == len(want_rows)
    if len(want_rows):
        assert np.array_equal(_np(rows).reshape(-1, t), want_rows)
    # count tables: S_i = GF table of g_i..g_d
    Sh = S.cpu().numpy().astype(np.uint64)
    for i in range(len(g)):
        assert np.array_equal(Sh[i], corc.gf_table(top - 1, g[i:])), i
    assert np.array_equal(Sh[len(g)], (np.arange(top) == 0).astype(np.uint64))


@pytest.mark.parametrize("kat", [k for k in read_golden_csv("memo_kats.csv") if k["tier"] in ("small", "mid")],
                         ids=lambda k: f"{k['tail']}-{k['top']}")
def test_memo_kats(kat, corc):
    """Memo CSR hash vs SURVEY App. A KATs (incl. C3 t=3, 13.5 M rows, whole-grid fill)."""
    tail, top = parse_gens(kat["tail"]), int(kat["top"])
    memo = fz.memo_build((7,) + tail, len(tail), top)
    rows, _, _ = memo.views()
    assert memo.info["entries"] == int(kat["entries"])
    assert corc.hash_rows(_np(rows).reshape(-1, len(tail))) == int(kat["H"], 16)


# ---------------------------------------------------------------------- C1
def test_c1_all_m(corc):
    """C1: Z(m; 6,9,20) for every m <= 1000 from ONE memo (t=2, top 1001), bit-exact."""
    memo = fz.memo_build(C1_GENS, C1_T, C1_MAX_N + 1)
    tot, hs = 0, 0
    for m in range(C1_MAX_N + 1):
        out, rows, _ = fz.enumerate(memo, m, "materialize")
        want, cnt, h = corc.enumerate(m, C1_GENS)
        assert rows == cnt
        assert np.array_equal(_np(out).reshape(-1, 3)[:rows], want.reshape(-1, 3)), m
        tot += rows
        _, _, gh = fz.enumerate(memo, m, "hash")
        assert gh == h, m
        hs = (hs + gh) % (1 << 64)
        assert fz.count(memo, m) == cnt
    assert tot == 162781 and hs == 0x54C291A6F228CA38      # SURVEY App. A aggregate


# -------------------------------------------------------------- random suite
@pytest.mark.parametrize("seed", range(200))
def test_random_small(seed, corc):
    """random (d 2..5, g <= 25, n <= 120) instances, every t in 0..d-1,
    full memo (top n+1) and a larger top; list, count and hash bit-exact."""
    g, n, _ = random_instance(seed)
    want, cnt, h = corc.enumerate(n, g)
    for t in range(0, len(g)):
        for top in (n + 1, n + 37):
            memo = fz.memo_build(g, t, top)
            out, rows, _ = fz.enumerate(memo, n, "materialize")
            assert rows == cnt
            assert np.array_equal(_np(out).reshape(-1, len(g))[:rows], want.reshape(-1, len(g))), (t, top)
            assert fz.enumerate(memo, n, "hash")[1:] == (cnt, h)
            assert fz.enumerate(memo, n, "count")[1] == cnt
            assert fz.count(memo, n) == cnt


@pytest.mark.parametrize("seed", range(24))
def test_mid_sharded(seed, corc):
    """Mid-size Table-1-shaped instances spanning many slices with ragged tails; shard
    invariance over 1, 2, 3 and 7 shards (concatenation in rank order == the full list)."""
    g, n, t = random_instance_mid(seed)
    memo = fz.memo_build(g, t, n + 1)
    _check_materialize(memo, n, corc, g, shards=(1, 2, 3, 7))


# ------------------------------------------------------------------- Table 1
@pytest.mark.parametrize("d,md,n", TABLE1_ROWS, ids=lambda x: str(x))
def test_table1_rows(d, md, n, corc):
    """C5: every Table 1 row with the paper's memo_dim and a full memo
    (top = n+1): count == oracle (erratum R14 at line 318 -> 779257) and
    hash == oracle; rows element by element up to 3 M rows."""
    g = table1_gens(d)
    memo = fz.memo_build(g, md, n + 1)
    cnt, h = corc.count_hash(n, g, use_o2=True)
    out, rows, _ = fz.enumerate(memo, n, "materialize")
    assert rows == cnt
    assert fz.enumerate(memo, n, "hash")[1:] == (cnt, h)
    assert fz.enumerate(memo, n, "count")[1] == cnt
    got = _np(out).reshape(-1, d)[:rows]
    if cnt <= 3_000_000:
        want, _, _ = corc.enumerate(n, g, use_o2=True)
        assert np.array_equal(got, want)
    else:
        assert corc.hash_rows(got) == h      # host recomputation of the hash of the GPU list


# ---------------------------------------------------------------------- C2
def test_c2_full_materialize(corc):
    """C2 at full size in bench.py's launch configuration: 100 000 681 rows, element by element."""
    g, n, t = C2.gens, C2.n, C2.t
    memo = fz.memo_build(g, t, n + 1)
    out, rows, _ = fz.enumerate(memo, n, "materialize")
    want, cnt, h = corc.enumerate(n, g, use_o2=True)
    assert rows == cnt == 100_000_681
    assert np.array_equal(_np(out).reshape(-1, 4), want)
    assert h == 0x5FC4E1F53888C565
    assert fz.enumerate(memo, n, "hash")[1:] == (cnt, h)
    assert fz.enumerate(memo, n, "count")[1] == cnt


# ------------------------------------------- odd / non-multiple-of-4 d at 1e8 rows (word stream)
@pytest.mark.parametrize("d,n,t", [(6, 6748, 3), (9, 1966, 5), (9, 1966, 4)], ids=lambda x: str(x))
def test_large_materialize_odd_d(d, n, t, corc):
    """>= 1e8-row materialize at d = 6 and d = 9 (Table 1's generators, the first n with |Z(n)| >= 1e8) element
    by element against O2: rows leave through the 16-B word stream (d = 6 t = 3, d = 9 t = 5:
    >= 8 rows per leading prefix) or lane by lane (d = 9 t = 4: ~9 per prefix is at the threshold)."""
    from fzinputs import table1_gens

    g = table1_gens(d)
    want, cnt, h = corc.enumerate(n, g, use_o2=True)
    assert cnt >= 10**8
    memo = fz.memo_build(g, t, n + 1)
    out, rows, _ = fz.enumerate(memo, n, "materialize")
    assert rows == cnt
    assert np.array_equal(_np(out).reshape(-1, d)[:rows], want.reshape(-1, d))
    del out
    assert fz.enumerate(memo, n, "hash")[1:] == (cnt, h)


# ---------------------------------------------------------------------- C3
@pytest.mark.parametrize("t", (2, 3, 4))
def test_c3_count_hash(t, corc):
    """C3 count+hash: count == GF count, hash == SURVEY App. A KAT, identical for every t
    (t = 4: a 30.4 GB memo of 1.9e9 rows, above the default 8e9 B cap)."""
    if t == 4:
        fz.set_memo_cap(64 << 30)
    try:
        memo = fz.memo_build(C3_GENS, t, C3_N + 1)
    finally:
        fz.set_memo_cap(0)
    _, rows, h = fz.enumerate(memo, C3_N, "hash")
    assert rows == corc.gf_count(C3_N, C3_GENS) == 10_002_178_949
    assert h == 0xBE3AEBC0385B7792
    assert fz.enumerate(memo, C3_N, "count")[1] == rows


# ---------------------------------------------------------------------- C4
@pytest.mark.parametrize("t,walk", [(3, "runs"), (2, "runs"), (3, "pairs")])
def test_c4_count(t, walk, corc, monkeypatch):
    """C4 count-only, t = 3 (u16 card image) and t = 2 (u8 image, 6.14e12 lookups): the pair walk's count ==
    the independent GF count (3 356 809 984 741), whole and over 2 / 8 shards, in bench.py's launch
    configuration (BASELINE configs[3]); both COUNT kernels (k5_runs default, k5_pairs via FZ_COUNT_WALK)."""
    monkeypatch.setenv("FZ_COUNT_WALK", walk)
    memo = fz.memo_build(C4.gens, t, C4.n + 1, entries=False)
    want = corc.gf_count(C4.n, C4.gens)
    assert want == 3_356_809_984_741
    p = fz.Plan(memo, C4.n, "count")
    assert p.walk() == ("count_pairs" if walk == "pairs" else "count_staged", 2 if t == 3 else 1)
    p.launch()
    assert p.result()[0] == want
    assert fz.count(memo, C4.n) == want
    for k in (2, 8):
        tot = sum(fz.enumerate(memo, C4.n, "count", shard=s, nshards=k)[1] for s in range(k))
        assert tot == want, k


@pytest.mark.parametrize("walk", ["runs", "pairs"])
@pytest.mark.parametrize("seed", range(32))
def test_count_staged(seed, walk, corc, monkeypatch):
    """COUNT with the card table staged in shared memory, forced on small walks (FZ_COUNT_SMEM=2):
    the COUNT kernels for L >= 3 (k5_runs, k5_pairs) and the run-per-lane walk (L = 2) give the oracle's count, whole
    and cut into 2, 3 and 7 shards, for every t."""
    monkeypatch.setenv("FZ_COUNT_SMEM", "2")
    monkeypatch.setenv("FZ_COUNT_WALK", walk)
    for g, n in (random_instance(seed)[:2], random_instance_mid(seed)[:2]):
        cnt = corc.gf_count(n, g)
        for t in range(0, len(g)):
            memo = fz.memo_build(g, t, n + 1, entries=False)
            assert fz.enumerate(memo, n, "count")[1] == cnt, (g, n, t)
            for k in (2, 3, 7):
                assert sum(fz.enumerate(memo, n, "count", shard=s, nshards=k)[1] for s in range(k)) == cnt, (g, n, t, k)


def test_c4_shape_hash(corc):
    """C4-shaped hash pin (n = 10000): 251 416 858 rows, H from SURVEY App. A."""
    memo = fz.memo_build(C4.gens, 3, 10001)
    assert fz.enumerate(memo, 10000, "hash")[1:] == (251_416_858, 0x2C3F7155D27A609C)


# ----------------------------------------------------------------- edge cases
EDGE = [((6, 9, 20), 0, 2), ((6, 9, 20), 43, 2), ((6, 9, 20), 44, 1), ((2, 3), 1, 1), ((5,), 35, 0), ((5,), 36, 0),
        ((1, 1, 1), 50, 1), ((3, 3, 3), 30, 2), ((4, 6), 1000, 1), ((1,), 0, 0), ((7, 7), 700, 0),
        ((2, 4, 8, 16, 32, 64, 128, 256, 512, 1024), 300, 3)]


@pytest.mark.parametrize("g,n,t", EDGE, ids=lambda x: str(x))
def test_edges(g, n, t, corc):
    """n = 0, non-representable n, d = 1, g_i = 1, duplicates, gcd > 1, t = 0, d = 10."""
    memo = fz.memo_build(g, t, n + 1)
    _check_materialize(memo, n, corc, g, shards=(1, 3))


def test_errors():
    memo = fz.memo_build((6, 9, 20), 2, 101)
    with pytest.raises(fz.FzError) as e:
        fz.enumerate(memo, 101, "materialize")          # n >= top
    assert e.value.status == 1
    out = torch.empty((3, 3), dtype=torch.int32, device="cuda")
    with pytest.raises(fz.FzError) as e:
        fz.enumerate(memo, 100, "materialize", out=out)  # |Z(100)| = 7 > 3 rows
    assert e.value.status == 4
    cm = fz.memo_build((6, 9, 20), 2, 101, entries=False)
    with pytest.raises(fz.FzError):
        fz.enumerate(cm, 100, "materialize")             # count-only memo


def test_run_host_end_to_end(corc):
    """fz_run_host (host buffers, chunked D2H) == oracle."""
    for g, n, t in (((13, 37, 38, 40), 5000, 2), ((6, 9, 20), 1000, 2), ((11, 13, 17, 19), 4000, 2)):
        want, cnt, h = corc.enumerate(n, g)
        host = torch.empty((cnt, len(g)), dtype=torch.int32).pin_memory()
        r, hh = fz.run_host(g, t, n, "materialize", host)
        assert r == cnt
        assert np.array_equal(host.numpy().view(np.uint32), want)
        assert fz.run_host(g, t, n, "hash") == (cnt, h)
        assert fz.run_host(g, t, n, "count")[0] == cnt


# ------------------------------------------- f3: output streamed through a bounded device ring
@pytest.mark.parametrize("ring", [1024, 4096, 1 << 20], ids=lambda r: f"ring{r}")
def test_run_host_ring_small(ring, corc):
    """fz_run_host streams MATERIALIZE output through a device ring
    of 4 slots (down to 256 B = 16-21 rows a slot: thousands of chunks, every slot reused many times),
    element by element == the oracle; the device workspace is memo + headers + ring, whatever |Z(n)|."""
    for g, n, t in (((13, 37, 38, 40), 5000, 2), ((6, 9, 20), 1000, 2), ((13, 37, 38, 40, 41), 1500, 3),
                    ((23, 29, 31), 3001, 1)):
        want, cnt, h = corc.enumerate(n, g, use_o2=True)
        nb = fz.run_workspace_bytes(g, t, n, "materialize", ring_bytes=ring)
        lay = fz.Layout(g, t, n + 1, memo_top=fz.MEMO_TOP_AUTO)
        assert nb <= lay.workspace_bytes + 4096 + max(ring, 4 * 256)     # bounded: not |Z(n)| * 4 d
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        host = torch.empty((max(cnt, 1), len(g)), dtype=torch.int32).pin_memory()
        r, hh = fz.run_host(g, t, n, "materialize", host, workspace=ws)
        assert r == cnt
        assert np.array_equal(host.numpy().view(np.uint32)[:cnt], want.reshape(-1, len(g))), (g, n, ring)


def test_run_host_ring_c2(corc):
    """C2's 1.6 GB output streams through a 64 MB device ring (workspace < 128 MB) into pinned host memory,
    element by element == O2 (BASELINE configs[1])."""
    g, n, t = C2.gens, C2.n, C2.t
    nb = fz.run_workspace_bytes(g, t, n, "materialize", ring_bytes=64 << 20)
    assert nb < (128 << 20)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    want, cnt, h = corc.enumerate(n, g, use_o2=True)
    host = torch.empty((cnt, len(g)), dtype=torch.int32).pin_memory()
    r, _ = fz.run_host(g, t, n, "materialize", host, workspace=ws)
    assert r == cnt == 100_000_681
    assert np.array_equal(host.numpy().view(np.uint32), want.reshape(-1, len(g)))
    assert fz.run_host(g, t, n, "hash", workspace=ws) == (cnt, h)


# ------------------------------------------------------- f1: full DP table (t = d)
def test_full_table_c1(corc):
    """t = d builds Alg 2/3's whole table F[m], m <= 1000; every
    Z(m) is then a table block.  Second GPU route for C1; table == Alg 2 row by row."""
    g, N = C1_GENS, C1_MAX_N
    memo = fz.memo_build(g, len(g), N + 1)
    rows, off, _ = memo.views()
    want_rows, want_off = corc.memo_alg2(g, N + 1)
    assert np.array_equal(off.cpu().numpy().astype(np.uint64), want_off)
    assert np.array_equal(_np(rows).reshape(-1, 3), want_rows)
    tot, hs = 0, 0
    for m in (0, 1, 43, 44, 500, 999, 1000):
        out, r, _ = fz.enumerate(memo, m, "materialize")
        want, cnt, h = corc.enumerate(m, g)
        assert r == cnt and np.array_equal(_np(out).reshape(-1, 3)[:r], want.reshape(-1, 3))
        assert fz.enumerate(memo, m, "hash")[1:] == (cnt, h)
        assert fz.enumerate(memo, m, "count")[1] == cnt
    for m in range(N + 1):
        _, r, h = fz.enumerate(memo, m, "hash")
        tot += r
        hs = (hs + h) % (1 << 64)
    assert tot == 162781 and hs == 0x54C291A6F228CA38


@pytest.mark.parametrize("seed", range(40))
def test_full_table_random(seed, corc):
    g, n, _ = random_instance(seed)
    memo = fz.memo_build(g, len(g), n + 1)
    want, cnt, h = corc.enumerate(n, g)
    for ns in (1, 3):
        parts, hs = [], 0
        for s in range(ns):
            out, r, _ = fz.enumerate(memo, n, "materialize", shard=s, nshards=ns)
            parts.append(_np(out).reshape(-1, len(g))[:r])
            hs = (hs + fz.enumerate(memo, n, "hash", shard=s, nshards=ns)[2]) % (1 << 64)
        got = np.concatenate(parts)
        assert np.array_equal(got, want.reshape(-1, len(g))) and hs == h


@pytest.mark.parametrize("mode", ["materialize", "count", "hash"])
def test_device_plan_matches_host_cut(mode):
    """K4 cuts shards on the device; fz_layout_shard_rows makes the same cut on the host."""
    g, n, t = (13, 37, 38, 40, 41), 3000, 2
    lay = fz.Layout(g, t, n + 1)
    memo = fz.Memo(layout=lay)
    for ns in (1, 2, 5, 8):
        rb, rl = lay.shard_rows(n, mode, ns)
        for s in range(ns):
            p = fz.Plan(memo, n, mode, s, ns)
            assert (p.row_begin, p.rows) == (rb[s], rl[s]), (mode, ns, s)


# --------------------------------------------- f2: partial memo (topOfMemo <= n)
@pytest.mark.parametrize("seed", range(60))
def test_partial_random(seed, corc):
    """memo rows only for x < memo_top <= n.  Every t in 1..d and
    several memo_top: the list == O1 and == Alg 5 run with the same topOfMemo (the paper's Else
    branch), hash and count bit-exact, shard invariance over 1 and 3 shards."""
    g, n, _ = random_instance(seed)
    want, cnt, h = corc.enumerate(n, g)
    for t in range(1, len(g) + 1):
        for mt in sorted({1, max(1, n // 3), max(1, n // 2 + 1), max(1, n)}):
            memo = fz.memo_build(g, t, n + 1, memo_top=mt)
            assert memo.info["memo_top"] == mt
            parts, hs = [], 0
            for ns in (1, 3):
                parts, hs = [], 0
                for s in range(ns):
                    out, r, _ = fz.enumerate(memo, n, "materialize", shard=s, nshards=ns)
                    parts.append(_np(out).reshape(-1, len(g))[:r])
                    hs = (hs + fz.enumerate(memo, n, "hash", shard=s, nshards=ns)[2]) % (1 << 64)
                got = np.concatenate(parts)
                assert np.array_equal(got, want.reshape(-1, len(g))), (t, mt, ns)
                assert hs == h, (t, mt, ns)
            assert fz.enumerate(memo, n, "count")[1] == cnt
            if t < len(g) and n <= 80 and seed % 4 == 0:
                alg5 = np.array(O.alg5_run(n, g, t, top=mt), dtype=np.uint32).reshape(-1, len(g))
                assert np.array_equal(got, alg5), (t, mt)


@pytest.mark.parametrize("tail,top,mt", [((9, 20), 1001, 400), ((17, 19), 30233, 9000), ((3, 5, 8), 500, 137),
                                         ((38, 40, 41, 42), 3001, 1500)], ids=lambda x: str(x))
def test_partial_memo_rows(tail, top, mt, corc):
    """The partial memo holds exactly Alg 2's F[0..memo_top-1] (CSR) while the count tables cover
    every x < top."""
    g = (5,) + tuple(tail)
    memo = fz.memo_build(g, len(tail), top, memo_top=mt)
    rows, off, S = memo.views()
    want_rows, want_off = corc.memo_alg2(tail, mt)
    assert memo.info["entries"] == len(want_rows)
    assert np.array_equal(_np(rows).reshape(-1, len(tail)), want_rows)
    assert np.array_equal(off.cpu().numpy().astype(np.uint64)[:mt + 1], want_off)
    Sh = S.cpu().numpy().astype(np.uint64)
    for i in range(len(g)):
        assert np.array_equal(Sh[i], corc.gf_table(top - 1, g[i:])), i


@pytest.mark.parametrize("frac", [0.5, 0.9])
def test_partial_c2(frac, corc):
    """C2 with a partial memo (memo_top = frac * n), in bench.py's launch configuration: 100 000 681
    rows element by element against O2, hash == SURVEY App. A."""
    g, n, t = C2.gens, C2.n, C2.t
    memo = fz.memo_build(g, t, n + 1, memo_top=int(frac * n))
    out, rows, _ = fz.enumerate(memo, n, "materialize")
    want, cnt, h = corc.enumerate(n, g, use_o2=True)
    assert rows == cnt == 100_000_681
    assert np.array_equal(_np(out).reshape(-1, 4), want)
    assert fz.enumerate(memo, n, "hash")[1:] == (cnt, 0x5FC4E1F53888C565)


def test_partial_auto_cap(corc):
    """memo_top = AUTO under a small cap: the largest memo_top whose rows fit, and the same rows."""
    g, n = (13, 37, 38, 40, 41), 3000
    full = fz.memo_build(g, 3, n + 1)
    cap = full.info["entries"] * 4 * 3 // 5
    fz.set_memo_cap(cap)
    try:
        memo = fz.memo_build(g, 3, n + 1, memo_top=fz.MEMO_TOP_AUTO)
        mt = memo.info["memo_top"]
        assert 1 <= mt <= n
        card = corc.gf_table(n, g[2:])
        assert memo.info["entries"] == int(card[:mt].sum()) and memo.info["entries"] * 12 <= cap
        assert (int(card[:mt + 1].sum())) * 12 > cap
        want, cnt, h = corc.enumerate(n, g)
        out, rows, _ = fz.enumerate(memo, n, "materialize")
        assert rows == cnt and np.array_equal(_np(out).reshape(-1, 5)[:rows], want)
        # the end-to-end host call goes partial instead of failing with FZ_ECAP
        assert fz.run_host(g, 3, n, "hash") == (cnt, h)
    finally:
        fz.set_memo_cap(0)


@pytest.mark.parametrize("d,md,n", [r for r in TABLE1_ROWS if r[2] <= 3000][:8], ids=lambda x: str(x))
def test_partial_table1(d, md, n, corc):
    """Table 1 generators with a memo to n/2 only: hash and count == oracle."""
    g = table1_gens(d)
    memo = fz.memo_build(g, md, n + 1, memo_top=n // 2 + 1)
    cnt, h = corc.count_hash(n, g, use_o2=True)
    assert fz.enumerate(memo, n, "hash")[1:] == (cnt, h)
    assert fz.enumerate(memo, n, "count")[1] == cnt


# ------------------------------------------------ slice kinds (row slices / walk-cost slices)
@pytest.mark.parametrize("beta,spw", [("0", "16"), ("1", "4"), ("16", "1"), ("16", "64"), ("200", "4")],
                         ids=lambda x: str(x))
@pytest.mark.parametrize("case", ["C2", "T95", "T1mid", "C3t3"])
def test_slice_kinds(case, beta, spw, corc, monkeypatch):
    """Both K5 slice kinds forced on workloads whose default is the other one: row slices (FZ_ROW_BETA=0) on
    short-round Table 1 walks, cost slices (beta 1..200 rows per visited prefix, 1..64 slices per warp) on C2 and
    C3: the same rows (element by element on a mid-size Table 1 walk), count and hash."""
    from fzinputs import table1_gens

    monkeypatch.setenv("FZ_ROW_BETA", beta)
    monkeypatch.setenv("FZ_SLICES_PER_WARP", spw)
    if case == "C2":
        g, n, t, kat = C2.gens, C2.n, C2.t, 0x5FC4E1F53888C565
    elif case == "C3t3":
        g, n, t, kat = C3_GENS, C3_N, 3, 0xBE3AEBC0385B7792
    elif case == "T95":
        g, n, t, kat = table1_gens(9), 1500, 5, None
    else:
        g, n, t, kat = table1_gens(8), 1200, 4, None
    memo = fz.memo_build(g, t, n + 1)
    _, rows, h = fz.enumerate(memo, n, "hash")
    if kat is None:
        cnt, kat = corc.count_hash(n, g, use_o2=True)
    else:
        cnt = corc.gf_count(n, g)
    assert (rows, h) == (cnt, kat)
    if case in ("T1mid", "T95"):
        out, rows, _ = fz.enumerate(memo, n, "materialize")
        got = _np(out).reshape(-1, len(g))[:rows]
        if case == "T1mid":
            want, _, _ = corc.enumerate(n, g, use_o2=True)
            assert np.array_equal(got, want)
        else:
            assert corc.hash_rows(got) == kat
