"""Strip sharding across ranks (parallel.py), exercised on CPU.

The device join per strip needs a GPU (see test_gpu_parity's strip test);
here the host logic is checked: strip planning, strip input selection, the
exactly-one-owner-strip property of every pair (with the CPU oracle), and the
single all_gather over a real 2-rank gloo process group.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1908_11740_b200 import parallel
from paper_1908_11740_b200.synth import make_config


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 0.02), (5, 0.02)])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_plan_strips_cover_rows(cfg, scale, world):
    r, s, k = make_config(cfg, scale)
    cuts = parallel.plan_strips(r, s, k, world)
    assert cuts[0] == 0 and cuts[-1] == k and len(cuts) == world + 1
    assert all(a < b for a, b in zip(cuts, cuts[1:]))


def test_plan_strips_balances_cost():
    r, s, k = make_config(2, 0.05)
    cuts = parallel.plan_strips(r, s, k, 4)
    w = parallel._row_entries(r, k) + parallel._row_entries(s, k)
    cost = parallel._row_cost(w, parallel._tile_counts(r, k), parallel._tile_counts(s, k))
    per = [cost[a:b].sum() for a, b in zip(cuts, cuts[1:])]
    assert max(per) / (sum(per) / 4) < 1.2
    ent = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
    assert max(ent) / (sum(ent) / 4) < 1.5  # equal-row strips give ~1.4 on cfg2


def test_row_cost_caps_giant_tiles():
    tr = np.array([[1000, 2], [0, 0]], dtype=np.int64)
    ts = np.array([[3000, 3], [5, 0]], dtype=np.int64)
    got = parallel._row_cost(np.array([10, 20], dtype=np.int64), tr, ts)
    cap = parallel.STRIP_CAP * 4000
    assert got.tolist() == [parallel.STRIP_KAPPA * 10 + cap + 6, parallel.STRIP_KAPPA * 20]


def _tile_rows(b, k):
    return parallel.row_range(b, k)


def test_strip_inputs_exact_selection():
    r, _, k = make_config(5, 0.02)
    for lo, hi in [(0, 10), (10, 500), (500, k), (0, k)]:
        sub = parallel.strip_inputs(r, k, lo, hi)
        r0, r1 = _tile_rows(r, k)
        want = np.nonzero((r1 >= lo) & (r0 < hi))[0]
        assert np.array_equal(sub[0], r[0][want])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_every_pair_owned_by_exactly_one_strip(world):
    """Union over strips of the pairs each strip owns = the full join, and the
    strips are disjoint: the oracle joined on each strip's inputs, filtered to
    owner rows inside the strip, reassembles the reference result."""
    r, s, k = make_config(1, 0.5)
    full = oracle.sorted_pairs(oracle.join(r, s, "2d", k)["pairs"])
    cuts = parallel.plan_strips(r, s, k, world)
    parts = []
    for lo, hi in zip(cuts, cuts[1:]):
        rr = parallel.strip_inputs(r, k, lo, hi)
        ss = parallel.strip_inputs(s, k, lo, hi)
        p = oracle.join(rr, ss, "2d", k)["pairs"]
        own = parallel.owner_rows(r, s, p, k)
        parts.append(p[(own >= lo) & (own < hi)])
    got = oracle.sorted_pairs(np.concatenate(parts))
    assert len(got) == len(full) and np.array_equal(got, full)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, counts, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = parallel.exchange_counts(counts[rank], 10 + rank, 20 + rank)
        tm = parallel.combine_counts(counts[rank], 10 + rank, 20 + rank, 0.5 + rank, world)
        out[rank] = (ex["pair_offset"], ex["pairs"], ex["a_r"], ex["a_s"], tm["t_max"])
    finally:
        dist.destroy_process_group()


def test_exchange_counts_gloo_two_ranks():
    world, port = 2, _free_port()
    counts = [7, 5]
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, counts, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0] == (0, 12, 21, 41, 1.5)
    assert res[1] == (7, 12, 21, 41, 1.5)


def _dist_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, s, k = make_config(1, 0.3)
        cuts = parallel.plan_strips(r, s, k, world)
        sl_r = tuple(torch.from_numpy(np.ascontiguousarray(a[rank::world])) for a in r)
        sl_s = tuple(torch.from_numpy(np.ascontiguousarray(a[rank::world])) for a in s)
        assert parallel.plan_strips_distributed(sl_r, sl_s, k) == cuts
        # self-join (s_cols=None): the same cost model on R alone
        r5, _, k5 = make_config(5, 0.01)
        sl5 = tuple(torch.from_numpy(np.ascontiguousarray(a[rank::world])) for a in r5)
        assert parallel.plan_strips_distributed(sl5, None, k5) == \
            parallel.plan_strips(r5, r5, k5, world)
        lo, hi = cuts[rank], cuts[rank + 1]
        got = {}
        for name, b in (("r", r), ("s", s)):
            # this rank's arbitrary input slice: every world-th rectangle
            sl = tuple(torch.from_numpy(np.ascontiguousarray(a[rank::world])) for a in b)
            mine = parallel.distribute(sl, k, cuts)
            got[name] = mine[0].numpy()
            want = parallel.strip_inputs(b, k, lo, hi)[0]
            assert np.array_equal(np.sort(got[name]), np.sort(want)), (rank, name)
        # strip join with the oracle, owner-row filter, then the pair gather
        rr = parallel.strip_inputs(r, k, lo, hi)
        ss = parallel.strip_inputs(s, k, lo, hi)
        p = oracle.join(rr, ss, "2d", k)["pairs"]
        own = parallel.owner_rows(r, s, p, k)
        p = torch.from_numpy(p[(own >= lo) & (own < hi)])
        ex = parallel.exchange_counts(len(p), 0, 0)
        allp = parallel.gather_pairs(p, ex, dst=0)
        if rank == 0:
            full = oracle.sorted_pairs(oracle.join(r, s, "2d", k)["pairs"])
            got_sorted = parallel.canonical_pairs(allp).numpy()
            out[rank] = bool(np.array_equal(got_sorted, full))
        else:
            out[rank] = allp is None
    finally:
        dist.destroy_process_group()


def test_distribute_and_gather_gloo_two_ranks():
    """Device-side input distribution (all_to_all) + pair gather, on 2 gloo
    ranks: each rank ends with exactly its strip's rectangles, and rank 0
    reassembles the reference pair list."""
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_dist_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res == {0: True, 1: True}


def test_tile_rows_torch_matches_host():
    r, _, k = make_config(5, 0.02)
    y0, y1 = parallel.tile_rows_torch(torch.from_numpy(r[3]), torch.from_numpy(r[4]), k)
    h0, h1 = parallel.row_range(r, k)
    assert np.array_equal(y0.numpy(), h0) and np.array_equal(y1.numpy(), h1)
