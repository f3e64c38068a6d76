"""Multi-process (world size 2, gloo, CPU) tests of the N > 1 host logic.

Each rank takes its shard from the library's host shard cut (the same cut the device planner K4
makes), computes its shard's {rows, hash} with the ORACLE (its row range of the oracle's list, hash
keyed by global row), and the ranks all_reduce(SUM) the 16-byte accumulator exactly as bench.py does
with NCCL on the GPU.  The reduced value must equal the oracle's whole-problem {count, hash}: this
checks that shards tile Z(n) in rank order, that the hash is additive under global row keys, and that
the u64 wrap survives the int64 collective.  No kernel runs here.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

# the last case has C4's shape (d = 8, generators 97..104, t = 3): its COUNT cut is the pair walk's cost cut
# (whole outer prefixes), the one bench.py's N > 1 headline (C4 count, one problem cut into N shards) uses
CASES = [((11, 13, 17, 19), 4000, 2), ((13, 37, 38, 40), 5000, 2), ((6, 9, 20), 1000, 2), ((13, 37, 38, 40, 41), 1000, 3),
         ((97, 98, 99, 100, 101, 102, 103, 104), 4500, 3)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_i64(u):
    return u - (1 << 64) if u >= (1 << 63) else u


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2407_20474_b200 import fz

    C = O.C()
    out = []
    for g, n, t in CASES:
        lay = fz.Layout(g, t, n + 1)
        for mode in ("materialize", "count"):
            rb, rl = lay.shard_rows(n, mode, world)
            rows, cnt, h = C.enumerate(n, g, use_o2=True)
            mine = rows[rb[rank]:rb[rank] + rl[rank]]
            hs = C.hash_rows(mine, row_base=rb[rank]) if len(mine) else 0
            acc = torch.tensor([len(mine), _to_i64(hs)], dtype=torch.int64)
            dist.all_reduce(acc, op=dist.ReduceOp.SUM)
            tot_rows = int(acc[0])
            tot_hash = int(acc[1]) & ((1 << 64) - 1)
            # shards tile [0, |Z|) in rank order
            ends = torch.tensor([rb[rank], rb[rank] + rl[rank]], dtype=torch.int64)
            gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(gathered, ends)
            tiles = all(int(gathered[i][1]) == int(gathered[i + 1][0]) for i in range(world - 1))
            out.append((g, n, mode, tot_rows == cnt, tot_hash == h, tiles, int(gathered[0][0]) == 0,
                        int(gathered[-1][1]) == cnt))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shard_cut_and_reduction_gloo(world):
    if not os.path.exists(os.path.join(ROOT, "paper_2407_20474_b200", "libfz.so")):
        pytest.fail("libfz.so missing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in res:
        for rec in out:
            assert all(rec[3:]), (rank, rec)


def test_count_cut_balances_prefixes():
    """COUNT shards cut the leading-prefix walk evenly; their row ranges still tile Z(n)."""
    from oracle import oracle as O
    from paper_2407_20474_b200 import fz

    g, n, t = (97, 98, 99, 100, 101, 102, 103, 104), 10000, 3
    lay = fz.Layout(g, t, n + 1, entries=False)
    rb, rl = lay.shard_rows(n, "count", 8)
    assert rb[0] == 0 and all(rb[i] + rl[i] == rb[i + 1] for i in range(7))
    assert rb[7] + rl[7] == O.C().gf_count(n, g)
    mrb, mrl = lay.shard_rows(n, "materialize", 8)
    assert max(mrl) - min(mrl) <= 1 and sum(mrl) == O.C().gf_count(n, g)
