"""Tile-row strip sharding across GPUs (one process per GPU).

The reference has no distributed execution; PBSM tiles are
independent join units, so the grid shards without any
data-path collective:

* ``plan_strips``  — cut the K tile rows into N contiguous strips whose
  per-row cost (|R|+|S| assignments plus capped per-tile pair tests) is
  balanced by a prefix sum;
* ``strip_inputs`` — the rectangles a rank needs: those whose tile-row range
  [tile_of(yl), tile_of(yu)] meets the strip (host-side distribution, before
  the timed window) — or, when every rank starts from its own slice of the
  inputs, ``distributed_join_slices``: a distributed strip plan (one
  all_reduce of per-row counts) and a device all_to_all (``distribute``);
* each rank runs the full pipeline restricted to its rows
  (``device.run_join(..., row_lo, row_hi)``); class labels use the GLOBAL
  tile_of, so a pair is emitted only in its global owner tile — no cross-rank
  duplicates, no candidate exchange;
* ``exchange_counts`` — the one collective: an all_gather of each rank's
  {pair_count, A_R, A_S}; its exclusive prefix gives the rank's global pair
  offset and the global result_count;
* ``gather_pairs`` / ``canonical_pairs`` — the pair shards on one rank, in
  lexicographic order when a canonical list is wanted.
"""

from __future__ import annotations

import numpy as np

__all__ = ["canonical_pairs", "combine_counts", "distribute", "distributed_join",
           "distributed_join_slices", "exchange_counts", "gather_pairs", "plan_strips",
           "plan_strips_distributed", "row_range", "strip_inputs", "strip_join"]


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


# Strip cost model (per tile row, integer so the host and the distributed
# plans agree exactly): KAPPA × entries + Σ_T min(|R_T|·|S_T|, CAP·(|R_T|+|S_T|))
# with the per-tile counts taken at each rectangle's lower-left tile.  Entries
# price the count / scatter / staging work (~47 ps each on one B200); the
# pair term prices the mini-join tests and output, which concentrate where
# both inputs pile up (cfg2: the clusters clipped onto y = 0 and y = 1 put 40%
# of all |R_T|·|S_T| in rows 0 and 1999).  Calibrated on the cfg2 strips
# timed one by one (tools/strip_emulation.py): ~1/2 entry per pair test; the
# cap stops the brute-forced giant tiles (~0.3 ps per test) from dominating.
STRIP_KAPPA = 2
STRIP_CAP = 256


def _row_cost(entries: np.ndarray, tr: np.ndarray, ts: np.ndarray) -> np.ndarray:
    """The cost model on per-row entries and (k, k) per-tile counts (numpy or torch)."""
    pairs = tr * ts
    cap = STRIP_CAP * (tr + ts)
    if isinstance(tr, np.ndarray):
        tests = np.minimum(pairs, cap)
    else:
        import torch

        tests = torch.minimum(pairs, cap)
    return STRIP_KAPPA * entries + tests.sum(1)


def _tile_counts(b, k: int) -> np.ndarray:
    """Rectangles per tile at their lower-left tile, (k, k) int64."""
    t = row_range(b, k)[0] * k + _tile_index(b[1], k)
    return np.bincount(t, minlength=k * k).reshape(k, k).astype(np.int64)


def plan_strips(r, s, k: int, world: int) -> list[int]:
    """Row cut points [0 = c_0 < ... < c_N = k] balancing the per-row cost
    (entries and capped pair tests, ``_row_cost``) by a prefix sum."""
    if world <= 1:
        return [0, k]
    if world > k:
        raise ValueError(f"cannot split {k} tile rows over {world} ranks")
    w_r = _row_entries(r, k)
    w = w_r + (w_r if s is r else _row_entries(s, k))
    tr = _tile_counts(r, k)
    ts = tr if s is r else _tile_counts(s, k)
    return _cut_rows(_row_cost(w, tr, ts), k, world)


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
    mine = torch.tensor([count, a_r, a_s], dtype=torch.int64)
    if device is not None and torch.device(device).type == "cuda":
        # staged through page-locked memory: an asynchronous copy, so the
        # exchange costs one host sync (the read of the gathered counts)
        mine = mine.pin_memory().to(device, non_blocking=True)
    elif device is not None:
        mine = mine.to(device)
    if world == 1:
        allv = mine.view(1, 3)
    else:
        allv = torch.empty((world, 3), dtype=torch.int64, device=device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(allv, mine, group=group)
        else:  # gloo (CPU ranks) has no all_gather_into_tensor
            dist.all_gather(list(allv.unbind(0)), mine, group=group)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return exchange_from_rows(allv.cpu().numpy().tolist(), rank)


def exchange_from_rows(rows, rank: int) -> dict:
    """Every rank's (pair_count, A_R, A_S) → this rank's global pair offset
    and the totals (the exclusive prefix of the pair counts)."""
    v = np.asarray(rows, dtype=np.int64).reshape(-1, 3)
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
    return strip_join(rr, ss, k, lo, hi, device, collect=collect)


def strip_join(rr, ss, k: int, row_lo: int, row_hi: int, device=None, collect: bool = True):
    """One rank's join of its strip from host arrays already split
    (``strip_inputs``; pinned arrays copy without staging): host→device,
    the strip pipeline, the count exchange.  Returns (DeviceJoinResult,
    exchange dict)."""
    from . import device as dev

    # coordinates first on a side stream, ids last (mapped after the join):
    # the strip pipeline overlaps the PCIe copy, as in engine.join
    rd, sd = dev.to_device_pipelined(rr, ss, device if device is not None else "cuda")
    res = dev.run_join(rd, sd, k, k, collect=collect, row_lo=row_lo, row_hi=row_hi)
    ex = exchange_counts(res.count, res.header["a_r"], res.header["a_s"], device=device)
    return res, ex


# ---------------------------------------------------------------- §8(f) next
def tile_rows_torch(yl, yu, k: int):
    """Exact first/last tile row of torch float64 tensors (any device): the
    same floor-then-nudge against the boundaries i/k as axis_tile_index
    (geometry.py:87-106); torch's float64 mul/div are correctly rounded."""
    import torch

    bounds = torch.arange(k + 1, dtype=torch.float64, device=yl.device) / k

    def idx(p):
        i = torch.clamp((p * k).to(torch.int64), 0, k - 1)
        while True:
            down = (i > 0) & (p < bounds[i])
            up = (i < k - 1) & (p >= bounds[torch.clamp(i + 1, max=k)])
            if not bool((down | up).any()):
                return i
            i = i - down.to(torch.int64) + up.to(torch.int64)

    return idx(yl), idx(yu)


def _route_host(cols, k: int, cuts):
    """Host mirror of pbsm_route_count / pbsm_route_pack for CPU-resident
    slices (gloo ranks without a GPU): the same destination-major SJB1
    records {id, x_l, y_l, x_u, y_u} and per-destination counts."""
    import torch

    ids, xl, xu, yl, yu = (c.numpy() for c in cols)
    r0, r1 = _tile_index(yl, k), _tile_index(yu, k)
    c = np.asarray(cuts, dtype=np.int64)
    g0 = np.searchsorted(c, r0, side="right") - 1
    g1 = np.searchsorted(c, r1, side="right") - 1
    world = len(cuts) - 1
    parts, counts = [], []
    for g in range(world):
        m = (g0 <= g) & (g1 >= g)
        rec = np.stack([ids[m], xl[m].view(np.int64), yl[m].view(np.int64),
                        xu[m].view(np.int64), yu[m].view(np.int64)], axis=1)
        parts.append(rec)
        counts.append(len(rec))
    return (torch.from_numpy(np.ascontiguousarray(np.concatenate(parts))).reshape(-1),
            counts)


def _route_device(cols, k: int, cuts):
    """The routing kernels (pbsm_route_count + pbsm_route_pack): one send
    buffer of destination-major 40-byte records and the per-destination
    counts (one small device→host read)."""
    import torch

    from . import _native
    from .device import _ptr, _raw_stream

    lib = _native.load()
    ids, xl, xu, yl, yu = cols
    n = len(ids)
    world = len(cuts) - 1
    dev = yl.device
    stream = _raw_stream(dev)
    cuts_d = torch.as_tensor(cuts, dtype=torch.int32).to(dev)
    scratch = torch.empty(int(lib.pbsm_route_scratch_bytes(n, k, world)), dtype=torch.uint8,
                          device=dev)
    dest = torch.empty(world, dtype=torch.int64, device=dev)
    _native.check(lib.pbsm_route_count(_ptr(yl), _ptr(yu), n, k, cuts_d.data_ptr(), world,
                                       scratch.data_ptr(), dest.data_ptr(), stream),
                  "pbsm_route_count")
    counts = dest.cpu().tolist()
    rec = torch.empty(5 * sum(counts), dtype=torch.int64, device=dev)
    _native.check(lib.pbsm_route_pack(_ptr(ids), _ptr(xl), _ptr(xu), _ptr(yl), _ptr(yu), n, k,
                                      cuts_d.data_ptr(), world, scratch.data_ptr(),
                                      _ptr(rec), stream), "pbsm_route_pack")
    return rec, counts


def _unpack(rec):
    """SJB1 records → (ids, xl, xu, yl, yu) columns (pbsm_unpack_records on
    the device, a strided view on the host)."""
    import torch

    n = rec.numel() // 5
    if not rec.is_cuda:
        r = rec.view(n, 5)
        f = r[:, 1:].contiguous().view(torch.float64)
        return (r[:, 0].contiguous(), f[:, 0].contiguous(), f[:, 2].contiguous(),
                f[:, 1].contiguous(), f[:, 3].contiguous())
    from . import _native
    from .device import _ptr, _raw_stream
    from .errors import DatasetError

    lib = _native.load()
    cols = [torch.empty(n, dtype=torch.int64, device=rec.device)] + [
        torch.empty(n, dtype=torch.float64, device=rec.device) for _ in range(4)]
    bad = torch.empty(1, dtype=torch.int32, device=rec.device)
    _native.check(lib.pbsm_unpack_records(_ptr(rec), n, *(_ptr(c) for c in cols),
                                          bad.data_ptr(), _raw_stream(rec.device)),
                  "pbsm_unpack_records")
    if n and int(bad.item()):  # (routed records were validated rectangles: a bug guard)
        raise DatasetError("distribute: a received record has a lower bound above its upper")
    return tuple(cols)


def distribute(cols, k: int, cuts, group=None):
    """Device-side input distribution.

    Every rank holds an arbitrary slice of one input as (ids, xl, xu, yl, yu)
    tensors; afterwards every rank holds exactly the rectangles whose tile-row
    range meets its strip [cuts[rank], cuts[rank+1]) — a rectangle spanning a
    strip boundary goes to every strip it touches, as the strip join needs.
    The routing kernels pack the slice destination-major into one buffer of
    40-byte records (pbsm_route_count / pbsm_route_pack); then one all_to_all
    of the per-destination counts and ONE all_to_all_single of the packed
    records (NCCL over NVLink on GPUs; gloo on CPU ranks, which pack with the
    host mirror ``_route_host``), and the receiver unpacks the records into
    columns (pbsm_unpack_records)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if len(cuts) != world + 1:
        raise ValueError(f"{len(cuts) - 1} strips for {world} ranks")
    rec, sc = (_route_device if cols[0].is_cuda else _route_host)(cols, k, cuts)
    send_counts = torch.as_tensor(sc, dtype=torch.int64).to(rec.device)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc = recv_counts.tolist()
    buf = torch.empty(5 * sum(rc), dtype=torch.int64, device=rec.device)
    dist.all_to_all_single(buf, rec, [5 * c for c in rc], [5 * c for c in sc], group=group)
    return _unpack(buf)


def _cut_rows(w, k: int, world: int) -> list[int]:
    """The cut rule of plan_strips on a per-row entry vector."""
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


def plan_strips_distributed(r_cols, s_cols, k: int, group=None) -> list[int]:
    """plan_strips when every rank holds only a slice of R and S: per-row
    entry counts and per-tile counts of the local slices (torch, on the
    slices' device), one all_reduce, then the same cost model and cut rule —
    every rank gets identical cuts."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world <= 1:
        return [0, k]
    if world > k:
        raise ValueError(f"cannot split {k} tile rows over {world} ranks")
    dev = r_cols[0].device
    d = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    tiles = []
    for cols in ((r_cols,) if s_cols is None else (r_cols, s_cols)):
        _, xl, xu, yl, yu = cols
        c0, c1 = tile_rows_torch(xl, xu, k)
        r0, r1 = tile_rows_torch(yl, yu, k)
        span = c1 - c0 + 1
        d.scatter_add_(0, r0, span)
        d.scatter_add_(0, r1 + 1, -span)
        tiles.append(torch.bincount(r0 * k + c0, minlength=k * k).to(torch.int64))
    if s_cols is None:
        d *= 2
    # one all_reduce: per-row entry deltas and both inputs' per-tile counts
    buf = torch.cat([d] + tiles)
    dist.all_reduce(buf, group=group)
    w = torch.cumsum(buf[:k], 0)
    tr = buf[k + 1:k + 1 + k * k].view(k, k)
    ts = tr if s_cols is None else buf[k + 1 + k * k:].view(k, k)
    w = _row_cost(w, tr, ts).cpu().numpy()
    return _cut_rows(w, k, world)


def distributed_join_slices(r_cols, s_cols, k: int, collect: bool = True, group=None):
    """Strip-sharded join when each rank starts from an arbitrary slice of R
    and S already on its GPU (e.g. its shard of a file): distributed strip
    plan, device all_to_all of the inputs, local strip join, count exchange.
    ``s_cols=None`` is a self-join.  Returns (DeviceJoinResult, exchange)."""
    import torch.distributed as dist

    from . import device as dev

    rank = dist.get_rank(group)
    cuts = plan_strips_distributed(r_cols, s_cols, k, group)
    lo, hi = cuts[rank], cuts[rank + 1]
    rd = dev.DeviceRects(*distribute(r_cols, k, cuts, group))
    sd = rd if s_cols is None else dev.DeviceRects(*distribute(s_cols, k, cuts, group))
    res = dev.run_join(rd, sd, k, k, collect=collect, row_lo=lo, row_hi=hi)
    ex = exchange_counts(res.count, res.header["a_r"], res.header["a_s"],
                         device=rd.device, group=group)
    ex["cuts"] = cuts
    return res, ex


def gather_pairs(pairs, exchange: dict, dst: int = 0, group=None):
    """Pair gather (the reference concatenates its
    workers' chunks, engine.py:293-300): the ranks' pair shards land on rank
    `dst` only, each at its global pair offset (the exchange's prefix), by
    point-to-point sends straight into the output — no padding, nothing sent
    to the other ranks.  Returns the (P, 2) tensor on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = exchange["per_rank_pairs"]
    if len(pairs) != counts[rank]:
        raise ValueError(f"rank {rank}: {len(pairs)} pairs, the exchange says {counts[rank]}")
    # (gloo moves host memory only: device shards go through the host there)
    via_host = pairs.is_cuda and dist.get_backend(group) != "nccl"
    if rank != dst:
        if counts[rank]:
            dist.send(pairs.contiguous().cpu() if via_host else pairs.contiguous(),
                      dist.get_global_rank(group, dst) if group is not None else dst,
                      group=group)
        return None
    offs = np.concatenate([[0], np.cumsum(counts)])
    out = torch.empty((int(offs[-1]), 2), dtype=torch.int64,
                      device="cpu" if via_host else pairs.device)
    out[offs[rank]:offs[rank + 1]] = pairs.cpu() if via_host else pairs
    ops = [dist.P2POp(dist.irecv, out[offs[g]:offs[g + 1]],
                      dist.get_global_rank(group, g) if group is not None else g, group=group)
           for g in range(world) if g != rank and counts[g]]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return out.to(pairs.device) if via_host else out


def canonical_pairs(pairs):
    """(r_id, s_id) pairs in lexicographic order (the parity form; the
    reference's own list is unordered, engine.py:61-62).  Device tensors:
    the hand-written LSD radix sort (pbsm_sort_pairs, ``device.sort_pairs``);
    host tensors (gloo ranks): numpy's lexsort."""
    import torch

    if len(pairs) == 0:
        return pairs
    if pairs.is_cuda:
        from .device import sort_pairs

        return sort_pairs(pairs)
    p = pairs.numpy()
    return torch.from_numpy(p[np.lexsort((p[:, 1], p[:, 0]))])
