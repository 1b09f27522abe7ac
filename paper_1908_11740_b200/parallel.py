"""Tile-row strip sharding across GPUs (one process per GPU).

The reference has no distributed execution; PBSM tiles are
independent join units, so the grid shards without any
data-path collective:

* ``plan_strips``  — cut the K tile rows into N contiguous strips whose
  per-row entry counts (|R|+|S| assignments) are balanced by a prefix sum;
* ``strip_inputs`` — the rectangles a rank needs: those whose tile-row range
  [tile_of(yl), tile_of(yu)] meets the strip (host-side distribution, before
  the timed window; a device all-to-all is SURVEY §8(f) rank 1);
* each rank runs the full pipeline restricted to its rows
  (``device.run_join(..., row_lo, row_hi)``); class labels use the GLOBAL
  tile_of, so a pair is emitted only in its global owner tile — no cross-rank
  duplicates, no candidate exchange;
* ``exchange_counts`` — the one collective: an all_gather of each rank's
  {pair_count, A_R, A_S}; its exclusive prefix gives the rank's global pair
  offset and the global result_count.
"""

from __future__ import annotations

import numpy as np

__all__ = ["combine_counts", "exchange_counts", "plan_strips", "row_range", "strip_inputs"]


def _tile_index(p: np.ndarray, k: int) -> np.ndarray:
    """Vectorised axis_tile_index (geometry.py:87-106) with the exact i/k nudges."""
    i = np.clip((p * k).astype(np.int64), 0, k - 1)
    bounds = np.arange(k + 1, dtype=np.int64) / k
    while True:
        down = (i > 0) & (p < bounds[i])
        up = (i < k - 1) & (p >= bounds[np.minimum(i + 1, k)])
        if not (down.any() or up.any()):
            return i
        i = i - down + up


def row_range(b, k: int):
    """(first, last) tile row of every rectangle of one input."""
    return _tile_index(b[3], k), _tile_index(b[4], k)


def _row_entries(b, k: int) -> np.ndarray:
    """Assignments per tile row: Σ over rectangles of their column span."""
    c0, c1 = _tile_index(b[1], k), _tile_index(b[2], k)
    r0, r1 = row_range(b, k)
    span = (c1 - c0 + 1).astype(np.int64)
    d = np.zeros(k + 1, dtype=np.int64)
    np.add.at(d, r0, span)
    np.add.at(d, r1 + 1, -span)
    return np.cumsum(d[:k])


def plan_strips(r, s, k: int, world: int) -> list[int]:
    """Row cut points [0 = c_0 < ... < c_N = k] balancing per-row entries."""
    if world <= 1:
        return [0, k]
    if world > k:
        raise ValueError(f"cannot split {k} tile rows over {world} ranks")
    w_r = _row_entries(r, k)
    w = w_r + (w_r if s is r else _row_entries(s, k))
    cum = np.cumsum(w)
    total = cum[-1]
    cuts = [0]
    for g in range(1, world):
        c = int(np.searchsorted(cum, total * g / world, side="left")) + 1
        c = max(c, cuts[-1] + 1)             # non-empty strips
        c = min(c, k - (world - g))           # leave a row for each later strip
        cuts.append(c)
    cuts.append(k)
    return cuts


def strip_inputs(b, k: int, row_lo: int, row_hi: int):
    """Rectangles whose tile rows meet [row_lo, row_hi) (all of them if full grid)."""
    if row_lo == 0 and row_hi == k:
        return b
    r0, r1 = row_range(b, k)
    m = (r1 >= row_lo) & (r0 < row_hi)
    return tuple(np.ascontiguousarray(a[m]) for a in b)


def exchange_counts(count: int, a_r: int, a_s: int, device=None, group=None) -> dict:
    """All-gather {pair_count, A_R, A_S}; returns this rank's global pair offset
    and the global totals.  Uses the default process group (NCCL on GPUs,
    gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mine = torch.tensor([count, a_r, a_s], dtype=torch.int64, device=device)
    if world == 1:
        allv = mine.view(1, 3)
    else:
        allv = torch.empty((world, 3), dtype=torch.int64, device=device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(allv, mine, group=group)
        else:  # gloo (CPU ranks) has no all_gather_into_tensor
            dist.all_gather(list(allv.unbind(0)), mine, group=group)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    v = allv.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(v[:, 0])])
    return {"pair_offset": int(offs[rank]), "pairs": int(offs[-1]),
            "a_r": int(v[:, 1].sum()), "a_s": int(v[:, 2].sum()),
            "per_rank_pairs": v[:, 0].tolist()}


def combine_counts(count: int, a_r: int, a_s: int, t_local: float, world: int,
                   device=None) -> dict:
    """exchange_counts + the max over ranks of the timed region (bench only)."""
    import torch
    import torch.distributed as dist

    out = exchange_counts(count, a_r, a_s, device=device)
    t = torch.tensor([t_local], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["t_max"] = float(t.item())
    return out


def owner_rows(r, s, pairs: np.ndarray, k: int) -> np.ndarray:
    """Tile row that owns each (r_id, s_id) pair: the row of max(r.yl, s.yl)
    (Eq. 1's reference point, geometry.py:64-72).  Ids must be row indices."""
    yl = np.maximum(r[3][pairs[:, 0]], s[3][pairs[:, 1]])
    return _tile_index(yl, k)


def distributed_join(r, s, k: int, device=None, collect: bool = True):
    """One rank's share of a strip-sharded K×K join (call under torchrun).

    Every rank plans the same strips, keeps the rectangles meeting its strip,
    joins its tile rows on its GPU and learns its global pair offset from the
    single all_gather.  Returns (DeviceJoinResult, exchange dict)."""
    import torch.distributed as dist

    from . import device as dev

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    cuts = plan_strips(r, s, k, world)
    lo, hi = cuts[rank], cuts[rank + 1]
    rr = strip_inputs(r, k, lo, hi)
    ss = rr if s is r else strip_inputs(s, k, lo, hi)
    rd = dev.to_device(rr, device)
    sd = rd if s is r else dev.to_device(ss, device)
    res = dev.run_join(rd, sd, k, k, collect=collect, row_lo=lo, row_hi=hi)
    ex = exchange_counts(res.count, res.header["a_r"], res.header["a_s"], device=device)
    return res, ex
