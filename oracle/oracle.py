"""CPU ORACLE for Z(n) = {a in N^d : sum a_i g_i = n}.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_2407_20474_b200`` never imports it and shares no code
with it; this module never imports the product package.

Contents (each function cites the passage it follows):

* ``brute_force``      -- O0: every vector with a_i <= n/g_i, filtered by phi = n,
                          sorted descending (bruteForceFactorizations).
* ``enum_py``          -- O1 in pure Python, the nested-loop definition (
                          order: PAPER.md:120-134, reading R1 = descending lex).
* ``alg1_sets``        -- PAPER.md:93-108, Algorithm FactorizationsUpToElement with the
                          relaxed bounds of PAPER.md:112-113 (sets, unordered).
* ``alg2_lists``       -- PAPER.md:139-153, Algorithm LexicographicFactorizationListsUpToElement.
* ``alg3_cardinalities`` -- PAPER.md:171-192, the cardinality bookkeeping of
                          LexFacListsUpToElement_FactorizationwiseParallel with the C[0]
                          reading R5.
* ``next_candidate`` / ``next_candidate_dynamic`` / ``alg5_run`` -- PAPER.md:203-222,
                          PAPER.md:238-265, PAPER.md:271-288 (single stream, readings R6-R11).
* ``gf_count_py``      -- |Z(n)| = [x^n] prod 1/(1-x^{g_i}) (coin-change DP, Python ints).
* ``d2_count``         -- closed form for d = 2.
* ``hash_row`` / ``hash_list`` -- reading R17, the build's order-sensitive hash.
* ``C``                -- ctypes wrapper of ``liboracle.so`` (fz_oracle.c): O1/O2 at scale,
                          GF count (u128), Alg 2 memo.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from math import gcd

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
MASK64 = (1 << 64) - 1


# --------------------------------------------------------------------- O0 / O1
def brute_force(n: int, g: tuple[int, ...]) -> list[tuple[int, ...]]:
    """O0: all a with a_i <= n // g_i and sum a_i g_i = n, sorted
    descending lexicographically (reading R1)."""
    ranges = [range(n // gi + 1) for gi in g]
    sols = [a for a in itertools.product(*ranges) if sum(x * y for x, y in zip(a, g)) == n]
    return sorted(sols, reverse=True)


def enum_py(n: int, g: tuple[int, ...]) -> list[tuple[int, ...]]:
    """O1: nested loops, each a_k from floor(rem/g_k) down to 0, the last
    coordinate solved by divisibility.  Descending loops => descending lex."""
    d = len(g)
    out: list[tuple[int, ...]] = []

    def rec(k: int, rem: int, prefix: tuple[int, ...]) -> None:
        if k == d - 1:
            if rem % g[k] == 0:
                out.append(prefix + (rem // g[k],))
            return
        for a in range(rem // g[k], -1, -1):
            rec(k + 1, rem - a * g[k], prefix + (a,))

    rec(0, n, ())
    return out


# ------------------------------------------------------------------ Alg 1 / 2 / 3
def alg1_sets(n: int, g: tuple[int, ...]) -> dict[int, set[tuple[int, ...]]]:
    """PAPER.md:93-108 FactorizationsUpToElement, relaxed to m in [0,n], m-g_i >= 0
    (PAPER.md:112-113).  Returns F[m] as sets, F[0] = {0}."""
    d = len(g)
    F: dict[int, set[tuple[int, ...]]] = {0: {(0,) * d}}
    for m in range(1, n + 1):
        Z: set[tuple[int, ...]] = set()
        for i in range(d):
            if m - g[i] >= 0:
                Z |= {a[:i] + (a[i] + 1,) + a[i + 1:] for a in F[m - g[i]]}
        F[m] = Z
    return F


def incr(a: tuple[int, ...], i: int) -> tuple[int, ...]:
    """PAPER.md:61-68 incr_i (0-based i here)."""
    return a[:i] + (a[i] + 1,) + a[i + 1:]


def is_all_zeroes_left_of_index(a: tuple[int, ...], i: int) -> bool:
    """PAPER.md:148 isAllZeroesLeftOfIndex (0-based i: a_j = 0 for all j < i)."""
    return all(x == 0 for x in a[:i])


def alg2_lists(n: int, g: tuple[int, ...], top: int | None = None) -> list[list[tuple[int, ...]]]:
    """PAPER.md:139-153 LexicographicFactorizationListsUpToElement.  F[0] = [0] is the
    base case and the m-loop starts at 1 (reading R3b); returns F[0..top-1]
    (top defaults to n+1)."""
    d = len(g)
    top = n + 1 if top is None else top
    F: list[list[tuple[int, ...]]] = [[(0,) * d]]
    for m in range(1, top):
        Z: list[tuple[int, ...]] = []
        for i in range(d):
            if m - g[i] >= 0:
                Z += [incr(a, i) for a in F[m - g[i]] if is_all_zeroes_left_of_index(a, i)]
        F.append(Z)
    return F


def alg3_cardinalities(n: int, g: tuple[int, ...]) -> tuple[list[list[tuple[int, ...]]], list[list[int]]]:
    """PAPER.md:171-192 LexFacListsUpToElement_FactorizationwiseParallel, executed
    sequentially: per (m, i) startIndex = sum_{j<i} C[m-g_i][j],
    count = sum_{j>=i} C[m-g_i][j], copy-and-increment the source slice, record C[m][i].
    C[0] = (0,...,0,1) (reading R5; the printed [1,...,1] contradicts the footnote
    at PAPER.md:166)."""
    d = len(g)
    Z: list[list[tuple[int, ...]]] = [[(0,) * d]]
    C: list[list[int]] = [[0] * (d - 1) + [1]]
    for m in range(1, n + 1):
        Zm: list[tuple[int, ...]] = []
        Cm = [0] * d
        for i in range(d):
            if m - g[i] >= 0:
                src = m - g[i]
                start = sum(C[src][:i])
                cnt = sum(C[src][i:])
                Zm += [incr(a, i) for a in Z[src][start:start + cnt]]
                Cm[i] = cnt
        Z.append(Zm)
        C.append(Cm)
    return Z, C


# ------------------------------------------------------- Alg N / Alg 4 / Alg 5
def phi(a, g) -> int:
    """PAPER.md:201 phi(a) = sum_i a_i g_i."""
    return sum(x * y for x, y in zip(a, g))


def set_initial_candidate(n: int, g: tuple[int, ...]) -> dict:
    """Reading R8: a = (ceil(n/g_1), 0, ..., 0), wasValid = (g_1 | n)."""
    d = len(g)
    a = [-(-n // g[0])] + [0] * (d - 1)
    return {"a": a, "b": [0] * d, "wasValid": n % g[0] == 0, "endOfStream": False}


def next_candidate(st: dict, n: int, g: tuple[int, ...]) -> None:
    """PAPER.md:203-222 nextCandidate, steps 1-12 (rightmost-nonzero loop over
    j in 1..d-1, reading R7).  In place."""
    if st["endOfStream"]:
        return
    a, d = st["a"], len(g)
    i = -1
    for j in range(d - 1):                   # excluding the final (R7)
        if a[j] > 0:
            i = j
    if i < 0:
        st["endOfStream"] = True
        st["wasValid"] = False      # reading R9b: a step that ends at step 3 yields no candidate
        return
    a[d - 1] = 0
    a[i] -= 1
    p = n - phi(a, g)
    m, r = divmod(p, g[i + 1])
    st["wasValid"] = True
    if r != 0:
        m += 1
        st["wasValid"] = False
    a[i + 1] = m
    if tuple(a) <= tuple(st["b"]):
        st["endOfStream"] = True


def next_candidate_dynamic(st: dict, n: int, g: tuple[int, ...], memo: list, memo_dim: int,
                           top: int) -> list[tuple[int, ...]]:
    """PAPER.md:238-265 nextCandidateDynamic.  p = n - phi(a) is computed right
    after the decrement (reading R6); memo condition i = d - memoDim and
    p < topOfMemo (strict, R10).  Returns the step's Outputs."""
    outputs: list[tuple[int, ...]] = []
    if st["endOfStream"]:
        return outputs
    a, d = st["a"], len(g)
    i = -1
    for j in range(d - 1):
        if a[j] > 0:
            i = j
    if i < 0:
        st["endOfStream"] = True
        st["wasValid"] = False      # reading R9b
        return outputs
    a[d - 1] = 0
    a[i] -= 1
    p = n - phi(a, g)
    if i + 1 == d - memo_dim and p < top:          # 1-based i = d - memoDim
        lead = tuple(a[: d - memo_dim])
        outputs = [lead + tuple(e) for e in memo[p]]
        st["wasValid"] = False
    else:
        m, r = divmod(p, g[i + 1])
        st["wasValid"] = True
        if r != 0:
            m += 1
            st["wasValid"] = False
        a[i + 1] = m
    if tuple(a) <= tuple(st["b"]):
        st["endOfStream"] = True
    return outputs


def alg5_run(n: int, g: tuple[int, ...], memo_dim: int, top: int | None = None,
             trace: list | None = None) -> list[tuple[int, ...]]:
    """PAPER.md:271-288 FactorizationsParallelLexicographicWithMemoization for one
    stream (W = 1; splitWork is prior work, reading R18): populateMemo (Alg 2 over the
    tail generators), setInitialCandidate, then loop nextCandidateDynamic
    + copyOutputsToBufferAndClear (valid candidate first, then Outputs)."""
    d = len(g)
    if d == 1:
        return [(n // g[0],)] if n % g[0] == 0 else []
    top = n + 1 if top is None else top
    memo = alg2_lists(max(top - 1, 0), tuple(g[d - memo_dim:]), top=top)
    st = set_initial_candidate(n, g)
    buf: list[tuple[int, ...]] = []
    if st["wasValid"]:
        buf.append(tuple(st["a"]))
    while not st["endOfStream"]:
        outs = next_candidate_dynamic(st, n, g, memo, memo_dim, top)
        if trace is not None:
            trace.append((tuple(st["a"]), st["wasValid"], tuple(outs)))
        if st["wasValid"]:
            buf.append(tuple(st["a"]))
        buf += outs
    return buf


# ------------------------------------------------------------- counts / hash
def gf_count_py(n: int, g: tuple[int, ...]) -> int:
    """Coefficient of x^n in prod 1/(1 - x^{g_i}): c[0] = 1; for g: c[x] += c[x-g]."""
    c = [0] * (n + 1)
    c[0] = 1
    for gi in g:
        for x in range(gi, n + 1):
            c[x] += c[x - gi]
    return c[n]


def d2_count(n: int, a: int, b: int) -> int:
    """Closed form |Z(n; a, b)|: 0 if gcd does not divide n, else
    floor(R/(AB)) + [A * ((R * A^{-1}) mod B) <= R mod AB], A=a/c, B=b/c, R=n/c."""
    c = gcd(a, b)
    if n % c:
        return 0
    A, B, R = a // c, b // c, n // c
    x0 = 0 if B == 1 else (R * pow(A, -1, B)) % B
    return R // (A * B) + (1 if A * x0 <= R % (A * B) else 0)


def _fmix64(x: int) -> int:
    x ^= x >> 33
    x = (x * 0xFF51AFD7ED558CCD) & MASK64
    x ^= x >> 33
    x = (x * 0xC4CEB9FE1A85EC53) & MASK64
    x ^= x >> 33
    return x


def hash_row(k: int, a) -> int:
    """Reading R17: order-sensitive row hash keyed by global row k."""
    x = ((k + 1) * 0x9E3779B97F4A7C15) & MASK64
    for v in a:
        x = ((x ^ int(v)) * 0xBF58476D1CE4E5B9) & MASK64
        x ^= x >> 29
    return _fmix64(x ^ len(a))


def hash_list(rows, row_base: int = 0) -> int:
    """H = sum_k h(row_base + k, f_k) mod 2^64 (R17)."""
    return sum(hash_row(row_base + k, r) for k, r in enumerate(rows)) & MASK64


# --------------------------------------------------------------- C oracle
class _COracle:
    """ctypes wrapper of oracle/liboracle.so (built by build_oracle())."""

    def __init__(self, path: str):
        L = ctypes.CDLL(path)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.orc_enum_o1.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, u32p, ctypes.c_uint64, u64p, u64p]
        L.orc_count_hash.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_uint64, ctypes.c_uint64, u64p, u64p]
        L.orc_gf_count.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, u64p, u64p]
        L.orc_gf_table.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, u64p]
        L.orc_memo_alg2.argtypes = [u32p, ctypes.c_int, ctypes.c_uint64, u32p, ctypes.c_uint64, u64p]
        L.orc_hash_row.argtypes = [ctypes.c_uint64, u32p, ctypes.c_int]
        L.orc_hash_row.restype = ctypes.c_uint64
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_hash_rows.argtypes = [u32p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64]
        L.orc_hash_rows.restype = ctypes.c_uint64
        self.L = L

    @staticmethod
    def _g(g):
        arr = np.ascontiguousarray(np.asarray(g, dtype=np.uint32))
        return arr, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))

    def enumerate(self, n: int, g, use_o2: bool = False, materialize: bool = True, cap: int | None = None):
        """O1/O2 single-threaded.  Returns (rows uint32[count, d] or None, count, hash)."""
        garr, gp = self._g(g)
        d = len(garr)
        cnt, h = ctypes.c_uint64(), ctypes.c_uint64()
        if materialize:
            if cap is None:
                cap = self.gf_count(n, g)
            out = np.empty((max(cap, 1), d), dtype=np.uint32)
            rc = self.L.orc_enum_o1(gp, d, n, int(use_o2), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                    cap, ctypes.byref(cnt), ctypes.byref(h))
        else:
            out = None
            rc = self.L.orc_enum_o1(gp, d, n, int(use_o2), None, 0, ctypes.byref(cnt), ctypes.byref(h))
        if rc:
            raise ValueError(f"orc_enum_o1 rc={rc}")
        if out is not None:
            out = out[: min(cnt.value, cap)]
        return out, cnt.value, h.value

    def count_hash(self, n: int, g, use_o2: bool = True, threads: int = 0, a1_range=None):
        """O1/O2 count + hash, OpenMP over a_1 (0 threads = library default)."""
        garr, gp = self._g(g)
        lo, hi = (0, (1 << 64) - 1) if a1_range is None else a1_range
        cnt, h = ctypes.c_uint64(), ctypes.c_uint64()
        rc = self.L.orc_count_hash(gp, len(garr), n, int(use_o2), threads, lo, hi, ctypes.byref(cnt), ctypes.byref(h))
        if rc:
            raise ValueError(f"orc_count_hash rc={rc}")
        return cnt.value, h.value

    def gf_count(self, n: int, g) -> int:
        garr, gp = self._g(g)
        lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
        rc = self.L.orc_gf_count(gp, len(garr), n, ctypes.byref(lo), ctypes.byref(hi))
        if rc:
            raise ValueError(f"orc_gf_count rc={rc}")
        return (hi.value << 64) | lo.value

    def gf_table(self, N: int, g) -> np.ndarray:
        garr, gp = self._g(g)
        out = np.empty(N + 1, dtype=np.uint64)
        rc = self.L.orc_gf_table(gp, len(garr), N, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        if rc:
            raise ValueError(f"orc_gf_table rc={rc}")
        return out

    def memo_alg2(self, g, top: int):
        """Alg 2 over generators g for m in [0, top).  Returns (rows uint32[E, t], off uint64[top+1])."""
        garr, gp = self._g(g)
        t = len(garr)
        cap = int(sum(int(self.gf_count(m, g)) for m in range(top))) if top <= 64 else None
        if cap is None:
            tbl = self.gf_table(top - 1, g)
            cap = int(tbl.sum(dtype=np.uint64))
        rows = np.empty((max(cap, 1), t), dtype=np.uint32)
        off = np.empty(top + 1, dtype=np.uint64)
        rc = self.L.orc_memo_alg2(gp, t, top, rows.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), cap,
                                  off.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        if rc:
            raise ValueError(f"orc_memo_alg2 rc={rc}")
        return rows[: int(off[top])], off

    def hash_row(self, k: int, a) -> int:
        arr, p = self._g(a)
        return self.L.orc_hash_row(k, p, len(arr))

    def hash_rows(self, rows: np.ndarray, row_base: int = 0) -> int:
        """Sum of R17 row hashes of a uint32[count, d] array, keys from row_base."""
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        cnt, d = rows.shape
        return self.L.orc_hash_rows(rows.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), cnt, d, row_base)

    def max_threads(self) -> int:
        return self.L.orc_max_threads()


_C: _COracle | None = None


def build_oracle(force: bool = False) -> str:
    """Compile fz_oracle.c -> liboracle.so with gcc (plain C11, OpenMP)."""
    src = os.path.join(_HERE, "fz_oracle.c")
    so = os.path.join(_HERE, "liboracle.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fopenmp", "-shared", "-fPIC", "-o", so, src])
    return so


def C() -> _COracle:
    global _C
    if _C is None:
        _C = _COracle(build_oracle())
    return _C
