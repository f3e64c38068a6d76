"""Seeded, synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

This module holds NO arithmetic of the method (no counting, no enumeration, no
hashing): only the generator tuples, elements and memo dimensions of the
workloads, and a seeded PRNG that draws small random instances.  Both
``oracle/`` and ``paper_2407_20474_b200`` are fed from here; neither imports
the other.

Workload recipe:

* C1-C5 are the fixed tuples of BASELINE.json ``configs`` / SURVEY §8 (no
  randomness).  Their shape follows Table 1: clustered,
  similar-magnitude generators; C5 is Table 1 itself.
* Random parity instances follow SPEC.md:459: d in 2..5, g_i in 1..25,
  n in 0..120, drawn from ``random.Random(seed)``; duplicates, gcd > 1 and
  g_i = 1 are allowed (reading R2).  ``random_instance_mid`` draws larger
  cases (several kernel tiles and a ragged tail) with the same structure.
"""
from __future__ import annotations

import random
from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    gens: tuple[int, ...]
    n: int
    t: int          # memo dimension (trailing generators tabulated)
    mode: str       # "materialize" | "count" | "hash"


# C1: <6,9,20>, every m in [0, 1000], tail t=2 (BASELINE.json configs[0])
C1_GENS = (6, 9, 20)
C1_MAX_N = 1000
C1_T = 2

# C2: d=4 <11,13,17,19>, n = 30232 (first n with |Z| >= 1e8), materialized
C2 = Workload("C2", (11, 13, 17, 19), 30232, 2, "materialize")

# C3: d=6 <23,29,31,37,41,43>, n = 17350 (first n with |Z| >= 1e10), count + hash, t sweep
C3_GENS = (23, 29, 31, 37, 41, 43)
C3_N = 17350
C3_T_SWEEP = (2, 3, 4)

# C4: d=8 generators near 100, large n, count only, sharded (SURVEY §8 proposal)
C4 = Workload("C4", (97, 98, 99, 100, 101, 102, 103, 104), 40000, 3, "count")
C4_SMALL_N = 10000   # hash-pinnable C4-shape element

# C5: Table 1 rows: gens (13,37,38[,40..45]); (d, memo_dim, n)
TABLE1_GENS_ALL = (13, 37, 38, 40, 41, 42, 43, 44, 45)
TABLE1_ROWS = (
    (3, 1, 100000), (3, 1, 200000), (3, 1, 300000),
    (4, 2, 5000), (4, 2, 10000), (4, 2, 15000),
    (5, 2, 1000), (5, 2, 3000), (5, 2, 5000), (5, 2, 10000),
    (5, 3, 1000), (5, 3, 3000), (5, 3, 5000),
    (6, 3, 1000), (6, 3, 3000), (6, 3, 5000),
    (6, 4, 1000), (6, 4, 2000), (6, 4, 3000),
    (7, 4, 1000), (7, 4, 1500), (7, 4, 2000),
    (8, 4, 1000), (8, 4, 1500), (8, 4, 2000),
    (9, 4, 500), (9, 4, 1000), (9, 4, 1500),
    (9, 5, 500), (9, 5, 1000), (9, 5, 1500),
)


def table1_gens(d: int) -> tuple[int, ...]:
    return TABLE1_GENS_ALL[:d]


def random_instance(seed: int, d_range=(2, 5), g_max: int = 25, n_max: int = 120):
    """SPEC.md:459 random parity instance: (gens, n, t) from random.Random(seed)."""
    r = random.Random(seed)
    d = r.randint(*d_range)
    gens = tuple(r.randint(1, g_max) for _ in range(d))
    n = r.randint(0, n_max)
    t = r.randint(1, d - 1) if d >= 2 else 1
    return gens, n, t


def random_instance_mid(seed: int):
    """Mid-size instance: clustered generators like Table 1 (one small leading
    generator followed by a tight cluster), n sized so |Z| spans many kernel tiles
    with a ragged tail.  Returns (gens, n, t)."""
    r = random.Random(1_000_003 + seed)
    d = r.randint(3, 6)
    lead = r.randint(3, 15)
    base = r.randint(20, 60)
    gens = (lead,) + tuple(base + r.randint(0, 12) for _ in range(d - 1))
    n = r.randint(150, {3: 6000, 4: 2500, 5: 1200, 6: 700}[d])
    t = r.randint(1, d - 1)
    return gens, n, t
