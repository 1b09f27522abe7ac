"""Device-side join pipeline: torch owns the memory, libpbsm does the work.

``run_join`` drives the C ABI (include/pbsm.h) through the four subsystems:

  pbsm_init → pbsm_count(R), pbsm_count(S) → pbsm_plan → [header read #1]
  → pbsm_scatter(R), pbsm_scatter(S) → pbsm_join_count → [header read #2]
  → pbsm_join_emit (collect mode) → [header read #3: guard bits]

The header reads are the only host synchronisations: #1 sizes the tile lists
(A_R, A_S, like ``write_pass`` sizing its buffers from the count pass,
partition.py:186-199), #2 sizes the pair array from the counted total (the
count-then-emit writer).  Everything else is enqueued on one CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import KernelError

__all__ = ["DeviceRects", "DeviceJoinResult", "PhaseProbe", "release_buffers", "run_join",
           "partition_columns", "points_to_device", "sort_pairs", "tile_counts", "to_device",
           "to_device_pipelined"]


@dataclass
class DeviceRects:
    """One input on the GPU in the reference's SoA column order."""

    ids: torch.Tensor   # int64 [n]
    xl: torch.Tensor    # float64 [n]
    xu: torch.Tensor
    yl: torch.Tensor
    yu: torch.Tensor
    # set by to_device_pipelined: recorded on the copy stream once the four
    # coordinate columns / the ids have landed; run_join makes its stream
    # wait on them right before the first kernel that reads them
    coords_ready: object = None
    ids_ready: object = None
    # the last-landing id column is copied in equal row chunks: (chunk_rows,
    # [event per chunk]) — see staged_pairs_to_host
    id_chunks: object = None

    def __len__(self) -> int:
        return int(self.ids.shape[0])

    @property
    def device(self) -> torch.device:
        return self.ids.device

    def columns(self):
        return self.ids, self.xl, self.xu, self.yl, self.yu


def points_to_device(batch, device="cuda") -> DeviceRects:
    """The point columns of an ε-distance join — ids and the lower corners
    (xl, yl) of a ``RectBatch`` (engine.py:333-334) — on the GPU; the square
    around each point is computed inside the kernels (pbsm_count_points).
    ``xu`` / ``yu`` alias ``xl`` / ``yl`` and are never read."""
    cols = []
    for a, dt in ((batch.ids, torch.int64), (batch.xl, torch.float64), (batch.yl, torch.float64)):
        cols.append(_host_tensor(a, dt, True).to(device, non_blocking=True))
    ids, px, py = cols
    return DeviceRects(ids, px, px, py, py)


INT64_MAX = (1 << 63) - 1


def to_device(batch, device="cuda", pinned: bool = True) -> DeviceRects:
    """Copy a ``RectBatch`` (or 5-tuple of arrays) to the GPU."""
    cols = batch if isinstance(batch, (tuple, list)) else (
        batch.ids, batch.xl, batch.xu, batch.yl, batch.yu)
    out = []
    for a, dt in zip(cols, (torch.int64,) + (torch.float64,) * 4):
        t = torch.from_numpy(np.ascontiguousarray(a))
        if t.dtype != dt:
            t = t.to(dt)
        if pinned and t.numel() > 0:
            t = t.pin_memory()
        out.append(t.to(device, non_blocking=True))
    return DeviceRects(*out)


_copy_streams: dict = {}
# staged return of host-input joins: the last id column crosses PCIe in
# ID_GROUPS chunks when it has at least ID_CHUNK_MIN rows
ID_GROUPS = int(os.environ.get("PBSM_ID_GROUPS", 8))
STAGED = os.environ.get("PBSM_STAGED", "1") != "0"
ID_CHUNK_MIN = 1 << 20


def _host_tensor(a, dt, pinned: bool) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype != dt:
        t = t.to(dt)
    if pinned and t.numel() > 0 and not t.is_pinned():
        t = t.pin_memory()
    return t


def to_device_pipelined(r, s, device="cuda"):
    """Copy R and S (``RectBatch`` or 5-tuples) to the GPU on a side stream in
    the order the join reads them — R's coordinates, S's coordinates, then
    the ids — with an event after each group, so run_join's count passes
    start while the rest is still crossing PCIe (the host→device copy is
    most of an end-to-end join).  Returns (R, S) DeviceRects (S is R when
    s is r)."""
    device = torch.device(device)
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    cs = _copy_streams.get(device.index)
    if cs is None:
        cs = _copy_streams[device.index] = torch.cuda.Stream(device)
    batches = [r] if s is r else [r, s]
    cols = [b if isinstance(b, (tuple, list)) else (b.ids, b.xl, b.xu, b.yl, b.yu)
            for b in batches]
    dts = (torch.int64,) + (torch.float64,) * 4
    host = [[None] * 5 for _ in batches]
    dev_cols = [[None] * 5 for _ in batches]
    # every later allocation reuses only blocks whose last use is already
    # enqueued on the current stream: one wait covers them all
    cs.wait_stream(torch.cuda.current_stream(device))

    def put(j, q, lo=None, hi=None):
        # each column is prepared right before its copy, so the first bytes
        # start crossing PCIe after one column's preparation, not ten
        if host[j][q] is None:
            host[j][q] = _host_tensor(cols[j][q], dts[q], True)
            dev_cols[j][q] = torch.empty(host[j][q].shape, dtype=dts[q], device=device)
        h, d = host[j][q], dev_cols[j][q]
        if lo is None:
            d.copy_(h, non_blocking=True)
        else:
            d[lo:hi].copy_(h[lo:hi], non_blocking=True)

    out = []
    with torch.cuda.stream(cs):
        coord_ev = []
        for j in range(len(batches)):
            for q in range(1, 5):
                put(j, q)
            ev = torch.cuda.Event()
            ev.record(cs)
            coord_ev.append(ev)
        last = len(batches) - 1
        for j, cev in enumerate(coord_ev):
            chunks = None
            n = len(cols[j][0])
            # (a self-join's pairs need both ids from the one column: a group
            # waits for the later of two chunks, so the tail is not shorter —
            # measured on cfg5, not staged)
            if j == last and last == 1 and n >= ID_CHUNK_MIN:
                # the last id column in ID_GROUPS row chunks, an event each:
                # the pairs whose ids are complete go back while the rest
                # is still in flight (staged_pairs_to_host)
                rows = -(-n // ID_GROUPS)
                evs = []
                for a in range(0, n, rows):
                    put(j, 0, a, a + rows)
                    e = torch.cuda.Event()
                    e.record(cs)
                    evs.append(e)
                chunks = (rows, evs)
                iev = evs[-1]
            else:
                put(j, 0)
                iev = torch.cuda.Event()
                iev.record(cs)
            out.append(DeviceRects(*dev_cols[j], coords_ready=cev, ids_ready=iev,
                                   id_chunks=chunks))
    return (out[0], out[0]) if s is r else (out[0], out[1])


def _wait(ev, stream_obj) -> None:
    if ev is not None:
        stream_obj.wait_event(ev)


@dataclass
class DeviceJoinResult:
    count: int
    pairs: torch.Tensor | None          # int64 [P, 2] (r_id, s_id) on the device
    header: dict = field(default_factory=dict)
    times: dict = field(default_factory=dict)  # seconds per phase (CUDA events)
    tile_counts: tuple | None = None      # (cnt_r, cnt_s) device views when kept
    rows_pending: bool = False            # pairs still hold row indices (defer_map)


# Host-side state of the driver, every cache keyed by (device, stream) so
# joins enqueued concurrently — from several threads, on several streams or
# devices — never share a workspace, a list buffer, a side stream or a pinned
# header; the dicts themselves are guarded by _state_lock.
_state_lock = threading.RLock()
_ws_cache: dict = {}


def _workspace(lib, device, kx, ky, row_lo, row_hi, stream: int = 0) -> torch.Tensor:
    key = (str(device), stream)
    grid = (kx, ky, row_lo, row_hi)
    with _state_lock:
        ent = _ws_cache.get(key)
        if ent is not None and ent[0] == grid:
            return ent[1]
        nbytes = lib.pbsm_workspace_bytes(kx, ky, row_lo, row_hi)
        if nbytes < 0:
            raise KernelError(f"invalid grid {kx}x{ky} rows [{row_lo},{row_hi})")
        _ws_cache.pop(key, None)  # one grid workspace per (device, stream)
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
        _ws_cache[key] = (grid, ws)
        return ws


# Internal buffers of a join (the two tile lists, the join scratch), kept per
# device and reused by the next join when large enough: a fresh multi-GB
# allocation per join let the caching allocator fall back to cudaMalloc /
# cudaFree now and then, stalling the join for milliseconds.  The returned
# pair arrays are always fresh.  release_buffers() gives the memory back.
_buf_cache: dict = {}


def _raw_stream(device) -> int:
    """cudaStream_t of the current stream on ``device`` (the cheap accessor:
    torch.cuda.current_stream() builds a Stream object, ~2 µs per call)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return torch._C._cuda_getCurrentRawStream(idx)


def _buffer(device, name: str, shape: tuple, dtype, stream: int) -> torch.Tensor:
    n = 1
    for d in shape:
        n *= d
    # per (device, stream): joins enqueued on different streams never share
    key = (str(device), stream, name)
    with _state_lock:
        ent = _buf_cache.get(key)
        if ent is not None and ent[1] == shape and ent[0].dtype == dtype:
            return ent[2]  # the same view as last time
        buf = ent[0] if ent is not None else None
        if buf is None or buf.dtype != dtype or buf.numel() < n:
            _buf_cache.pop(key, None)
            del buf, ent  # the old block is free before the larger one is requested
            buf = torch.empty(max(n, 1), dtype=dtype, device=device)
        view = buf[:n].view(shape)
        _buf_cache[key] = (buf, shape, view)
        return view


def release_buffers() -> None:
    """Drop the cached tile lists, join scratch and grid workspaces."""
    with _state_lock:
        _buf_cache.clear()
        _ws_cache.clear()
        _plan_cache.clear()
        _graph_cache.clear()
        _fast.clear()


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None or t.numel() == 0 else t.data_ptr()


# messages of RectBatch.validate (geometry.py:166-177), raised in the same order:
# R before S, inverted before out-of-range
_VALIDATION = (
    (_native.ERR_INVERTED, "inverted rectangle: lower bound exceeds upper bound"),
    (_native.ERR_RANGE, "coordinates outside [0, 1]; normalize the datasets first"),
    (_native.ERR_INVERTED << 2, "inverted rectangle: lower bound exceeds upper bound"),
    (_native.ERR_RANGE << 2, "coordinates outside [0, 1]; normalize the datasets first"),
)
_VALIDATION_BITS = sum(b for b, _ in _VALIDATION)


_hdr_local = threading.local()


def _read_header(lib, ws, stream, allow=0) -> _native.Header:
    # into page-locked memory: a pageable destination would go through the
    # driver's staging copy on this (synchronising) path.  One buffer per
    # host thread: the read is synchronous, so a thread never has two in
    # flight, and concurrent joins on other threads have their own.
    buf = getattr(_hdr_local, "buf", None)
    if buf is None:
        buf = _hdr_local.buf = torch.empty(C.sizeof(_native.Header), dtype=torch.uint8,
                                           pin_memory=True)
    dst = C.cast(C.c_void_p(buf.data_ptr()), C.POINTER(_native.Header))
    _native.check(lib.pbsm_read_header(ws.data_ptr(), dst, stream), "pbsm_read_header")
    h = _native.Header.from_buffer_copy(C.string_at(buf.data_ptr(), C.sizeof(_native.Header)))
    for bit, msg in _VALIDATION:
        if h.error & bit:
            raise ValueError(msg)
    bad = h.error & ~allow & ~_VALIDATION_BITS
    if bad:
        raise KernelError(f"device guard: {_native.describe_error(bad)} "
                          "(partition write overflow check, partition.py:229-233)")
    return h


class PhaseProbe:
    """Records a CUDA event after every library call (per-kernel timing in bench.py)."""

    def __init__(self):
        self.marks: list[tuple[str, torch.cuda.Event]] = []

    def mark(self, name: str) -> None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((name, ev))

    def durations(self) -> dict:
        """Seconds per phase name, summed over repeats."""
        out: dict = {}
        for (_, a), (name, b) in zip(self.marks, self.marks[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b) / 1e3
        return out


def pair_capacity(h) -> int:
    """Initial pair-buffer size: the exact bound when affordable, else a
    generous estimate (the emit pass reports overflow and is re-run)."""
    return int(min(h.pair_bound, 2 * (h.list_r + h.list_s) + (1 << 20)))


# tile lists (64 B per entry) above this size are scattered through the
# row-band copy (pbsm_bin): measured on B200, random record writes over a
# multi-GB list run at ~1 TB/s, within an L2-sized window at ~4 TB/s
BIN_LIST_BYTES = int(os.environ.get("PBSM_BIN_BYTES", 1 << 30))


def _binned(total: int, n: int, bin_bytes: int | None) -> bool:
    """Whether a tile list of ``total`` entries from ``n`` rectangles goes
    through the row-band copy: the copy costs ~80 B per rectangle, so it pays
    only where the random record writes dominate — large lists and heavy
    replication (cfg4: 1.7 entries per rectangle; cfg2/cfg3/cfg5: 1.1-1.5,
    measured slower).  ``bin_bytes`` None = BIN_LIST_BYTES, 0 = always."""
    thresh = BIN_LIST_BYTES if bin_bytes is None else bin_bytes
    return 64 * total > thresh and (bin_bytes == 0 or total >= 1.6 * n)


def _binned_pair(list_r: int, list_s: int, n_r: int, n_s: int, bin_bytes: int | None,
                 split: bool) -> bool:
    """Whether either input goes through the row-band copy.  Compact nested
    entries (``split``) halve the scattered bytes without the copy: with
    BIN_LIST_BYTES' default they replace it (cfg4: 13.99 -> 12.94 ms,
    profiles/r02zx_cfg4_bin_split_ab.txt); an explicit ``bin_bytes`` keeps
    the row-band copy."""
    if not (_binned(list_r, n_r, bin_bytes) or _binned(list_s, n_s, bin_bytes)):
        return False
    return not (split and bin_bytes is None)


def _banded(lib, b: DeviceRects, side: int, wsp: int, grid, stream, ids_p) -> torch.Tensor:
    """Row-band copy of one input: n 40-byte records {id (or row), xl, xu, yl, yu}."""
    band = torch.empty((len(b), 5), dtype=torch.int64, device=b.device)
    _native.check(lib.pbsm_bin(ids_p, _ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu),
                               len(b), side, wsp, *grid, band.data_ptr(), stream), "pbsm_bin")
    return band


# Sizes of the last synchronous plan per join shape (grid, strip, input
# sizes, cost model): with a hit, run_join skips the host read of the plan
# header — lists, unit grids and the pair buffer use these sizes and the emit
# runs bounded (pbsm_join_emit_bounded); the final header read checks every
# size and a miss re-runs the join synchronously.
_plan_cache: dict = {}
DUAL = os.environ.get("PBSM_DUAL", "1") != "0"
# A self-join (s is r) is partitioned ONCE: side 0 is counted and scattered,
# its counters are copied over side 1's before the plan and the join reads the
# one list for both inputs — the reference partitions the array twice
# (engine.py:231-232) into two identical datasets (PBSM_SELF_ONCE=0: as the
# reference)
SELF_ONCE = os.environ.get("PBSM_SELF_ONCE", "1") != "0"
_side_streams: dict = {}


def _side_stream(device, stream: int):
    """The side stream paired with the launching stream ``stream`` (S's count
    and scatter run there, concurrent with R's)."""
    key = (device.index, stream)
    with _state_lock:
        st = _side_streams.get(key)
        if st is None:
            st = _side_streams[key] = torch.cuda.Stream(device)
        return st

SPECULATE = os.environ.get("PBSM_SPECULATE", "1") != "0"
# compact nested entries (pbsm_scatter_split / pbsm_join_emit_split): one
# 32-byte sector per nested-tile entry instead of a 64-byte record.  The
# scatter saves one scattered store per nested entry (cfg2: 545 -> 444 µs,
# cfg3 4.76 -> 3.92 ms) but each emitted pair then gathers its two ids by row
# (cfg2 join +35 µs, cfg3 +0.6 ms) — so it is used when the pairs are at most
# SPLIT_PAIR_RATIO per nested entry (the previous join of the shape tells:
# speculative sizes), or when the ids are still in flight anyway (every pair
# is mapped afterwards).
SPLIT = os.environ.get("PBSM_SPLIT", "1") != "0"
SPLIT_PAIR_RATIO = float(os.environ.get("PBSM_SPLIT_PAIR_RATIO", 1.0))


def _split_ok(collect, eps, binned, ordered, nest_r, nest_s, n_r, n_s, pairs_hint,
              late) -> bool:
    if not (SPLIT and collect and eps is None and not binned and not ordered
            and nest_r + nest_s > 0 and max(n_r, n_s) < (1 << 32)):
        return False
    if late:
        return True
    return pairs_hint is not None and pairs_hint <= SPLIT_PAIR_RATIO * (nest_r + nest_s)
# The unit pipeline (units.cuh) is parity-green but measured slower than the
# tile-list pipeline on every BASELINE config: opt-in only.
UNITS = os.environ.get("PBSM_UNITS", "0") == "1"
UNIT_TARGET = int(os.environ.get("PBSM_UNIT_TARGET", "-1"))
_uhdr_local = threading.local()


def _read_uheader(lib, ws, stream, allow=0) -> _native.UHeader:
    buf = getattr(_uhdr_local, "buf", None)
    if buf is None:
        buf = _uhdr_local.buf = torch.empty(C.sizeof(_native.UHeader), dtype=torch.uint8,
                                            pin_memory=True)
    dst = C.cast(C.c_void_p(buf.data_ptr()), C.POINTER(_native.UHeader))
    _native.check(lib.pbsm_read_uheader(ws.data_ptr(), dst, stream), "pbsm_read_uheader")
    h = _native.UHeader.from_buffer_copy(C.string_at(buf.data_ptr(), C.sizeof(_native.UHeader)))
    for bit, msg in _VALIDATION:
        if h.error & bit:
            raise ValueError(msg)
    bad = (h.error | h.jerror) & ~allow & ~_VALIDATION_BITS
    if bad:
        raise KernelError(f"device guard: {_native.describe_error(bad)} "
                          "(partition write overflow check, partition.py:229-233)")
    return h


def _uworkspace(lib, device, kx, ky, row_lo, row_hi, stream: int) -> torch.Tensor:
    key = (str(device), stream, "units")
    grid = (kx, ky, row_lo, row_hi)
    with _state_lock:
        ent = _ws_cache.get(key)
        if ent is not None and ent[0] == grid:
            return ent[1]
        nbytes = lib.pbsm_unit_workspace_bytes(kx, ky, row_lo, row_hi)
        if nbytes < 0:
            raise KernelError(f"unit pipeline: unsupported grid {kx}x{ky} [{row_lo},{row_hi})")
        _ws_cache.pop(key, None)
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
        _ws_cache[key] = (grid, ws)
        return ws


def _unit_slots(a_total: int, n_units: int) -> int:
    """Scratch slots for the unit join: every join-tile entry (<= A_R + A_S),
    a tile record per two small tiles (<= A/4), chunk descriptors and the
    per-unit 128-byte alignment."""
    return int(a_total + a_total // 4 + a_total // 512 + 16 * n_units + 1024)


def _run_units(lib, r: DeviceRects, s: DeviceRects, kx: int, ky: int, row_lo: int, row_hi: int,
               *, collect: bool, timing: bool, mark, defer_map: bool,
               exact: bool = False) -> DeviceJoinResult:
    """The unit pipeline (include/pbsm.h): init → cell counts (R and S on two
    streams) → unit map → [header read, first join of a shape only] → unit
    bins (two streams) → per-unit partition + nested mini-joins → deferred
    large tiles → header read.  Repeated shapes allocate from the previous
    join's sizes; any overflow (flagged on the device, nothing written out of
    bounds) re-runs the join with the exact sizes."""
    device = r.device
    stream = _raw_stream(device)
    ws = _uworkspace(lib, device, kx, ky, row_lo, row_hi, stream)
    wsp = ws.data_ptr()
    grid = (kx, ky, row_lo, row_hi)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timing else None
    if ev:
        ev[0].record()
    mark("start")
    _native.check(lib.pbsm_unit_init(wsp, *grid, stream), "pbsm_unit_init")
    mark("init")
    cur = (torch.cuda.current_stream(device)
           if r.coords_ready is not None or s.coords_ready is not None else None)
    late = r.ids_ready is not None and s.ids_ready is not None
    main_st = torch.cuda.current_stream(device)
    side_st = _side_stream(device, stream)
    dual = DUAL and cur is None

    def two(fn):
        """fn(side, batch, stream) for R then S; S on the side stream when dual."""
        if dual:
            fork = torch.cuda.Event()
            fork.record(main_st)
            side_st.wait_event(fork)
        for side, b in ((0, r), (1, s)):
            _wait(b.coords_ready, cur)
            fn(side, b, side_st.cuda_stream if (dual and side == 1) else stream)
        if dual:
            j = torch.cuda.Event()
            j.record(side_st)
            main_st.wait_event(j)

    two(lambda side, b, st: _native.check(
        lib.pbsm_unit_count(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), len(b), side, wsp,
                            *grid, st), "pbsm_unit_count"))
    mark("count")
    _native.check(lib.pbsm_unit_map(wsp, *grid, len(r), len(s), UNIT_TARGET, stream),
                  "pbsm_unit_map")
    mark("map")
    key = (str(device), stream, "units", *grid, len(r), len(s), s is r)
    guess = None if (exact or not SPECULATE) else _plan_cache.get(key)
    if guess is None:
        h = _read_uheader(lib, ws, stream)
        mark("header")
        a_tot = int(h.a_r + h.a_s)
        sizes = {"bin_r": max(int(h.bin_r), 1), "bin_s": max(int(h.bin_s), 1),
                 "slots": _unit_slots(a_tot, int(h.n_units)),
                 "units": max(int(h.n_units), 1),
                 "pairs": int(min(2 * a_tot + (1 << 20), 1 << 34))}
    else:
        sizes = guess
    if sizes["slots"] > 0xffffffff:
        raise KernelError("unit pipeline: more than 2^32 list slots; use pipeline='tiles'")
    bins = []

    def do_bin(side, b, st):
        cap = sizes["bin_r" if side == 0 else "bin_s"]
        buf = _buffer(device, f"ubin{side}", (int(lib.pbsm_unit_bin_bytes(cap)),), torch.uint8,
                      stream)
        bins.append((buf, cap))
        _native.check(lib.pbsm_unit_bin(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), len(b),
                                        side, wsp, *grid, buf.data_ptr(), cap, st),
                      "pbsm_unit_bin")

    two(do_bin)
    mark("bin")
    if ev:
        ev[1].record()
    scratch = _buffer(device, "uscratch", (int(lib.pbsm_unit_scratch_bytes(sizes["slots"])),),
                      torch.uint8, stream)
    ids_r = None if late else _ptr(r.ids)
    ids_s = None if late else _ptr(s.ids)
    (b0, c0), (b1, c1) = bins
    cap = sizes["pairs"] if collect else 0  # count-only: every chunk counts, none writes
    while True:
        pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=device)
        _native.check(lib.pbsm_unit_join(wsp, *grid, b0.data_ptr(), c0, b1.data_ptr(), c1,
                                         ids_r, ids_s, scratch.data_ptr(), sizes["slots"],
                                         sizes["units"], pairs.data_ptr(), cap, stream),
                      "pbsm_unit_join")
        mark("join")
        h2 = _read_uheader(lib, ws, stream, allow=_native.ERR_PAIR_OVERFLOW
                           | _native.ERR_SCATTER_OVERFLOW | _native.ERR_INTERNAL)
        mark("header2")
        structural = (h2.bin_r > c0 or h2.bin_s > c1 or h2.scratch_used > sizes["slots"]
                      or h2.n_units > sizes["units"]
                      or (h2.error | h2.jerror) & (_native.ERR_SCATTER_OVERFLOW
                                                   | _native.ERR_INTERNAL))
        if structural:
            if guess is None and not exact:
                raise KernelError(f"unit pipeline: sizes from the plan were exceeded "
                                  f"({_native.describe_error(h2.error | h2.jerror)})")
            # another input behind the same shape: redo it with the exact plan
            with _state_lock:
                _plan_cache.pop(key, None)
            return _run_units(lib, r, s, kx, ky, row_lo, row_hi, collect=collect,
                              timing=timing, mark=mark, defer_map=defer_map, exact=True)
        if h2.pairs <= cap or not collect:
            break
        cap = int(h2.pairs)  # the pair estimate was short: join again into an exact buffer
    count = int(h2.pairs)
    pairs = pairs[:count]
    with _state_lock:
        for k_ in [k_ for k_ in _plan_cache if k_[:3] == key[:3]]:
            del _plan_cache[k_]
        _plan_cache[key] = {"bin_r": max(int(h2.bin_r), 1), "bin_s": max(int(h2.bin_s), 1),
                            "slots": int(h2.scratch_used) + 1024,
                            "units": max(int(h2.n_units), 1),
                            "pairs": max(cap, 1) if collect else sizes["pairs"]}
    if late and not defer_map:
        _map_ids(lib, pairs, count, r, s, cur, stream)
    if ev:
        ev[2].record()
        ev[2].synchronize()
    hd = h2.as_dict()
    hd["list_r"], hd["list_s"] = int(h2.a_r), int(h2.a_s)
    res = DeviceJoinResult(count, pairs if collect else None, header=hd,
                           rows_pending=late and defer_map and collect)
    if ev:
        res.times = {"partition": ev[0].elapsed_time(ev[1]) / 1e3,
                     "join": ev[1].elapsed_time(ev[2]) / 1e3,
                     "total": ev[0].elapsed_time(ev[2]) / 1e3}
    return res


def _with_exchange(res: DeviceJoinResult, exchange: bool) -> DeviceJoinResult:
    """The eager path's count exchange (after its own header read)."""
    if exchange and "exchange" not in res.header:
        from .parallel import exchange_counts

        res.header["exchange"] = exchange_counts(res.count, res.header["a_r"],
                                                 res.header["a_s"], device=res_device(res))
    return res


def res_device(res: DeviceJoinResult):
    return res.pairs.device if res.pairs is not None else torch.device(
        "cuda", torch.cuda.current_device())


def run_join(r: DeviceRects, s: DeviceRects, kx: int, ky: int, *, collect: bool = True,
             row_lo: int = 0, row_hi: int | None = None, timing: bool = False,
             keep_counts: bool = False, probe: PhaseProbe | None = None,
             ordered: bool = False, nested_max: int = -1,
             bin_bytes: int | None = None, defer_map: bool = False,
             pipeline: str | None = None, sweep_min: int = -1,
             eps: float | None = None, graph: bool = False,
             exchange: bool = False) -> DeviceJoinResult:
    """Join two device-resident inputs over a ``kx × ky`` grid (rows [row_lo, row_hi)).

    Two device pipelines compute the same pair set: the tile-list pipeline
    below (the default) and the unit pipeline (``pipeline="units"`` or
    PBSM_UNITS=1, where ``pbsm_unit_supported``; not for the ordered emit,
    forced cost-model thresholds, the binned scatter or ``keep_counts``).

    ``probe`` (optional) gets an event after each library call, named after
    the phase that call ran: init, count, plan, header, scatter, join, header2.
    ``nested_max`` overrides the mini-join cost-model threshold (pbsm_plan);
    ``sweep_min``: large tiles with |R_T|*|S_T| above it are sorted and swept,
    the others brute-forced (pbsm_plan; -1 = default, 0 = sweep them all);
    ``ordered`` selects the look-back (unit-major) output placement;
    ``bin_bytes``: tile lists larger than this go through the row-band copy
    (pbsm_bin) before the scatter (default BIN_LIST_BYTES; 0 = always).
    ``defer_map``: with id columns still in flight (to_device_pipelined) the
    pairs are returned as row indices (``rows_pending``) for
    staged_pairs_to_host instead of being mapped here.
    ``graph``: repeated joins of the same device inputs (same tensors, same
    shape) replay the whole enqueue sequence — init, both counts, plan, both
    scatters, bounded emit, header publish — as one CUDA graph, then one
    host sync; the returned ``pairs`` is then a view of the graph's output
    buffer, valid until the next graphed join of the same inputs.
    ``exchange`` (strip-sharded joins, torch.distributed initialised): the
    one collective of the join — every rank's {pair_count, A_R, A_S} — lands
    in ``header["exchange"]`` (parallel.exchange_counts' dict).  On the graph
    path it is an all_gather of the device header inside the graph, before
    the single host read (no host round trip in between).
    ``eps``: ε-distance join (epsilon_distance_join, engine.py:326-353) —
    ``r``/``s`` hold points (``points_to_device``: xl, yl = px, py), each
    standing for its side-eps square; candidates are refined inside the
    mini-joins (pbsm_join_emit_eps), so the count is the refined count.
    """
    if graph and _fast and FAST_REPLAY and collect and not (timing or keep_counts or ordered or defer_map
                                            or exchange) \
            and probe is None and pipeline is None and eps is None and len(r) and len(s):
        res = _fast_replay(r, s, kx, ky, row_lo, ky if row_hi is None else row_hi, nested_max,
                           bin_bytes, sweep_min)
        if res is not None:
            return res
    res = _run_join_impl(r, s, kx, ky, collect=collect, row_lo=row_lo, row_hi=row_hi,
                         timing=timing, keep_counts=keep_counts, probe=probe, ordered=ordered,
                         nested_max=nested_max, bin_bytes=bin_bytes, defer_map=defer_map,
                         pipeline=pipeline, sweep_min=sweep_min, eps=eps, graph=graph,
                         exchange=exchange)
    return _with_exchange(res, exchange)


def _run_join_impl(r: DeviceRects, s: DeviceRects, kx: int, ky: int, *, collect: bool = True,
             row_lo: int = 0, row_hi: int | None = None, timing: bool = False,
             keep_counts: bool = False, probe: PhaseProbe | None = None,
             ordered: bool = False, nested_max: int = -1,
             bin_bytes: int | None = None, defer_map: bool = False,
             pipeline: str | None = None, sweep_min: int = -1,
             eps: float | None = None, graph: bool = False,
             exchange: bool = False) -> DeviceJoinResult:
    """run_join without the eager count exchange (see run_join)."""
    mark = probe.mark if probe is not None else (lambda name: None)
    lib = _native.load()
    if row_hi is None:
        row_hi = ky
    device = r.device
    if len(r) == 0 or len(s) == 0:
        empty = torch.empty((0, 2), dtype=torch.int64, device=device) if collect else None
        return DeviceJoinResult(0, empty)
    half = eps_sq = None
    if eps is not None:
        # squares computed in the kernels; their entries carry the points, and
        # no tile is sorted + swept (its sorted copy would not carry them)
        half, eps_sq = eps / 2.0, eps * eps
        sweep_min, bin_bytes, pipeline = INT64_MAX, INT64_MAX, "tiles"
    if (pipeline == "units" or (pipeline is None and UNITS)) and not ordered and not keep_counts \
            and nested_max == -1 and bin_bytes is None and sweep_min == -1 \
            and lib.pbsm_unit_supported(kx, ky, row_lo, row_hi) == 1:
        return _run_units(lib, r, s, kx, ky, row_lo, row_hi, collect=collect, timing=timing,
                          mark=mark, defer_map=defer_map)
    stream = _raw_stream(device)
    if graph and GRAPHS and probe is None and not timing and collect and not ordered \
            and not keep_counts and eps is None and not defer_map and SPECULATE \
            and r.coords_ready is None and s.coords_ready is None and r.ids_ready is None:
        key = (str(device), stream, kx, ky, row_lo, row_hi, len(r), len(s), s is r, nested_max,
               bin_bytes, sweep_min)
        guess = _plan_cache.get(key)
        if guess is not None and not _binned_pair(
                guess["list_r"], guess["list_s"], len(r), len(s), bin_bytes,
                _split_ok(True, None, False, False, guess["nested_r"], guess["nested_s"],
                          len(r), len(s), guess["count"], False)):
            res = _run_graphed(lib, r, s, kx, ky, row_lo, row_hi, key, guess, nested_max,
                               sweep_min, stream, exchange)
            if res is not None:
                return res
    ws = _workspace(lib, device, kx, ky, row_lo, row_hi, stream)
    wsp = ws.data_ptr()
    grid = (kx, ky, row_lo, row_hi)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timing else None
    if ev:
        ev[0].record()
    mark("start")
    _native.check(lib.pbsm_init(wsp, *grid, stream), "pbsm_init")
    mark("init")
    # (the Stream object only when there are copy events to wait on)
    cur = (torch.cuda.current_stream(device)
           if r.coords_ready is not None or s.coords_ready is not None else None)
    # ids still in flight (to_device_pipelined): the entries carry row
    # indices and the pair list is mapped to ids at the end (pbsm_map_ids),
    # so nothing before the final map waits for the id columns
    late = r.ids_ready is not None and s.ids_ready is not None
    # S's count and scatter run on a side stream, concurrent with R's: each
    # pass' tail (its last, partly filled wave of blocks) overlaps the other
    # input's pass (measured: cfg2 1.262 -> 1.253 ms, cfg5 0.783 -> 0.753 ms,
    # cfg3 8.65 -> 8.55 ms).  With host inputs still crossing PCIe the counts
    # stay on one stream, each behind its own copy event.
    main_st = side_st = None
    if DUAL:
        main_st = torch.cuda.current_stream(device)
        side_st = _side_stream(device, stream)
    same = SELF_ONCE and s is r and half is None and cur is None and r.ids_ready is None
    dual = DUAL and cur is None and not same
    if dual:
        fork = torch.cuda.Event()
        fork.record(main_st)
        side_st.wait_event(fork)
    for side, b in ((0, r), (1, s)):
        if same and side == 1:  # S's counters are R's
            cnt_r_v, cnt_s_v = _tile_count_views(ws, kx, ky, kx * (row_hi - row_lo))
            cnt_s_v.copy_(cnt_r_v, non_blocking=True)
            continue
        _wait(b.coords_ready, cur)
        st_ = side_st.cuda_stream if (dual and side == 1) else stream
        if half is not None:
            _native.check(lib.pbsm_count_points(_ptr(b.xl), _ptr(b.yl), len(b), side, half, wsp,
                                                *grid, st_), "pbsm_count_points")
        else:
            _native.check(lib.pbsm_count(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), len(b),
                                         side, wsp, *grid, st_), "pbsm_count")
    if dual:
        join_ev = torch.cuda.Event()
        join_ev.record(side_st)
        main_st.wait_event(join_ev)
    mark("count")
    counts = None
    if keep_counts:  # per-tile counts, before the plan turns them into cursor ends
        counts = tuple(v.clone() for v in _tile_count_views(ws, kx, ky, kx * (row_hi - row_lo)))
    _native.check(lib.pbsm_plan(wsp, *grid, nested_max, sweep_min, stream), "pbsm_plan")
    mark("plan")
    key = (str(device), stream, kx, ky, row_lo, row_hi, len(r), len(s), s is r, nested_max,
           bin_bytes, sweep_min)
    guess = _plan_cache.get(key) if (SPECULATE and collect and not ordered
                                     and not keep_counts and eps is None) else None
    if guess is None:
        h = _read_header(lib, ws, stream)
        mark("header")
        list_r, list_s = h.list_r, h.list_s
        nest_r, nest_s = h.nested_r, h.nested_s
    else:
        h = None
        list_r, list_s = guess["list_r"], guess["list_s"]
        nest_r, nest_s = guess["nested_r"], guess["nested_s"]

    lists = []
    split = _split_ok(collect, eps, False, ordered, nest_r, nest_s, len(r), len(s),
                      guess["count"] if guess is not None else None, late)
    binned = _binned_pair(list_r, list_s, len(r), len(s), bin_bytes, split)
    split = split and not binned
    dual_sc = DUAL and not binned and not same
    split_bufs = []
    if dual_sc:
        fork = torch.cuda.Event()
        fork.record(main_st)
        side_st.wait_event(fork)
    for side, b, total in ((0, r, list_r), (1, s, list_s)):
        if same and side == 1:  # one scatter: the join reads R's list for both inputs
            lists.append(lists[0])
            if split:
                split_bufs.append(split_bufs[0])
            mark("scatter")
            continue
        ent = _buffer(device, f"list{side}", (max(total, 1), 8), torch.int64,
                      stream)  # 64 B records
        ids_p = None if late else _ptr(b.ids)
        if half is not None:
            _native.check(lib.pbsm_scatter_points(ids_p, _ptr(b.xl), _ptr(b.yl), len(b), side,
                                                  half, wsp, *grid, ent.data_ptr(), total,
                                                  side_st.cuda_stream if (dual_sc and side)
                                                  else stream), "pbsm_scatter_points")
            if dual_sc and side == 1:
                join_ev = torch.cuda.Event()
                join_ev.record(side_st)
                main_st.wait_event(join_ev)
            if side == 1:
                mark("scatter")
            lists.append(ent)
            continue
        if split:
            n32 = max(nest_s if side else nest_r, 1)
            rec32 = _buffer(device, f"rec32_{side}", (n32, 4), torch.int64, stream)
            split_bufs.append((rec32, n32))
            _native.check(lib.pbsm_scatter_split(ids_p, _ptr(b.xl), _ptr(b.xu), _ptr(b.yl),
                                                 _ptr(b.yu), len(b), side, wsp, *grid,
                                                 ent.data_ptr(), total, rec32.data_ptr(), n32,
                                                 side_st.cuda_stream if (dual_sc and side)
                                                 else stream), "pbsm_scatter_split")
            if dual_sc and side == 1:
                join_ev = torch.cuda.Event()
                join_ev.record(side_st)
                main_st.wait_event(join_ev)
            if side == 1:
                mark("scatter")
            lists.append(ent)
            continue
        if dual_sc:
            _native.check(lib.pbsm_scatter(ids_p, _ptr(b.xl), _ptr(b.xu), _ptr(b.yl),
                                           _ptr(b.yu), len(b), side, wsp, *grid, ent.data_ptr(),
                                           total, side_st.cuda_stream if side else stream),
                          "pbsm_scatter")
            if side == 1:
                join_ev = torch.cuda.Event()
                join_ev.record(side_st)
                main_st.wait_event(join_ev)
                mark("scatter")
            lists.append(ent)
            continue
        if _binned(total, len(b), bin_bytes):
            band = _banded(lib, b, side, wsp, grid, stream, ids_p)
            mark("bin")
            _native.check(lib.pbsm_scatter_banded(band.data_ptr(), len(b), side, wsp, *grid,
                                                  ent.data_ptr(), total, stream),
                          "pbsm_scatter_banded")
            del band
        else:
            _native.check(lib.pbsm_scatter(ids_p, _ptr(b.xl), _ptr(b.xu), _ptr(b.yl),
                                           _ptr(b.yu), len(b), side, wsp, *grid, ent.data_ptr(),
                                           total, stream), "pbsm_scatter")
        mark("scatter")
        lists.append(ent)
    if ev:
        ev[1].record()

    rl, sl = lists
    if guess is not None:
        cap, cn, rest = guess["pairs"], guess["nested"], guess["other"]
        lcap, mtile = guess["large"], guess["max_huge"]
        scratch = _buffer(device, "scratch",
                          (int(lib.pbsm_join_scratch_bytes(cn + rest, lcap)),),
                          torch.uint8, stream)
        pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=device)
        mark("alloc")
        if split:
            _emit_split(lib, wsp, grid, rl, list_r, sl, list_s, split_bufs, r, s, late, None,
                        (cn, rest, lcap, mtile), scratch, pairs, cap, stream, guess["count"])
        else:
            _native.check(lib.pbsm_join_emit_bounded(wsp, *grid, rl.data_ptr(), list_r,
                                                     sl.data_ptr(), list_s, cn, rest, lcap,
                                                     mtile, scratch.data_ptr(), pairs.data_ptr(),
                                                     cap, stream), "pbsm_join_emit_bounded")
        mark("join")
        h2 = _read_header(lib, ws, stream,
                          allow=_native.ERR_PAIR_OVERFLOW | _native.ERR_SCATTER_OVERFLOW)
        mark("header2")
        if (h2.list_r > list_r or h2.list_s > list_s or h2.chunks_nested > cn
                or h2.chunks_sorted + h2.n_items > rest or h2.pairs > cap
                or (split and (h2.nested_r > nest_r or h2.nested_s > nest_s))
                or h2.error & (_native.ERR_PAIR_OVERFLOW | _native.ERR_SCATTER_OVERFLOW)):
            # another input behind the same shape: redo it with the exact plan
            with _state_lock:
                _plan_cache.pop(key, None)
            return run_join(r, s, kx, ky, collect=collect, row_lo=row_lo, row_hi=row_hi,
                            timing=timing, keep_counts=keep_counts, probe=probe,
                            ordered=ordered, nested_max=nested_max, bin_bytes=bin_bytes,
                            defer_map=defer_map, pipeline="tiles", sweep_min=sweep_min, eps=eps)
        count = int(h2.pairs)
        if late and not defer_map:
            _map_ids(lib, pairs, count, r, s, cur, stream)
        if ev:
            ev[2].record()
            ev[2].synchronize()
        res = DeviceJoinResult(count, pairs[:count], header=h2.as_dict(),
                               rows_pending=late and defer_map)
        if ev:
            res.times = {"partition": ev[0].elapsed_time(ev[1]) / 1e3,
                         "join": ev[1].elapsed_time(ev[2]) / 1e3,
                         "total": ev[0].elapsed_time(ev[2]) / 1e3}
        return res

    n_units = h.n_units
    scratch = _buffer(device, "scratch",
                      (int(lib.pbsm_join_scratch_bytes(n_units, h.large_r + h.large_s)),),
                      torch.uint8, stream)
    pairs = None
    if not collect:
        if eps_sq is not None:
            _native.check(lib.pbsm_join_count_eps(wsp, *grid, rl.data_ptr(), sl.data_ptr(),
                                                  C.byref(h), scratch.data_ptr(), eps_sq, stream),
                          "pbsm_join_count_eps")
        else:
            _native.check(lib.pbsm_join_count(wsp, *grid, rl.data_ptr(), sl.data_ptr(),
                                              C.byref(h), scratch.data_ptr(), stream),
                          "pbsm_join_count")
        mark("join")
        h2 = _read_header(lib, ws, stream)
        mark("header2")
        count = int(h2.pairs)
    else:
        cap = pair_capacity(h)
        while True:
            pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=device)
            if eps_sq is not None:
                _native.check(lib.pbsm_join_emit_eps(wsp, *grid, rl.data_ptr(), sl.data_ptr(),
                                                     C.byref(h), scratch.data_ptr(),
                                                     pairs.data_ptr(), cap, int(ordered), eps_sq,
                                                     stream), "pbsm_join_emit_eps")
            elif split:
                _emit_split(lib, wsp, grid, rl, list_r, sl, list_s, split_bufs, r, s, late,
                            C.byref(h), (-1, -1, 0, 0), scratch, pairs, cap, stream)
            else:
                _native.check(lib.pbsm_join_emit(wsp, *grid, rl.data_ptr(), sl.data_ptr(),
                                                 C.byref(h), scratch.data_ptr(), pairs.data_ptr(),
                                                 cap, int(ordered), stream), "pbsm_join_emit")
            mark("join")
            h2 = _read_header(lib, ws, stream, allow=_native.ERR_PAIR_OVERFLOW)
            mark("header2")
            count = int(h2.pairs)
            if count <= cap:
                break
            cap = count  # rare: the estimate was short, emit again into an exact buffer
        pairs = pairs[:count]
        if late and not defer_map:
            _map_ids(lib, pairs, count, r, s, cur, stream)
        if not ordered and not keep_counts and eps is None:
            with _state_lock:
                for k_ in [k_ for k_ in _plan_cache if k_[:2] == key[:2]]:
                    del _plan_cache[k_]  # one shape per (device, stream)
                _plan_cache[key] = {"list_r": h.list_r, "list_s": h.list_s, "pairs": cap,
                                "nested": h.chunks_nested,
                                "other": h.chunks_sorted + h.n_items,
                                "large": int(h.large_r + h.large_s),
                                "max_huge": int(h.max_huge),
                                "nested_r": int(h.nested_r), "nested_s": int(h.nested_s),
                                "count": count}
    if ev:
        ev[2].record()
        ev[2].synchronize()
    res = DeviceJoinResult(count, pairs, header=h2.as_dict(),
                           rows_pending=late and defer_map and pairs is not None)
    if ev:
        res.times = {"partition": ev[0].elapsed_time(ev[1]) / 1e3,
                     "join": ev[1].elapsed_time(ev[2]) / 1e3,
                     "total": ev[0].elapsed_time(ev[2]) / 1e3}
    res.tile_counts = counts
    return res


def sort_pairs(pairs: torch.Tensor) -> torch.Tensor:
    """(n, 2) int64 device pairs → a new tensor in lexicographic (r_id, s_id)
    order: the stable LSD radix sort of pbsm_sort_pairs over the digits that
    vary (one small histogram read decides which)."""
    lib = _native.load()
    n = int(pairs.shape[0])
    out = pairs.contiguous().clone()
    if n <= 1:
        return out
    device = pairs.device
    stream = _raw_stream(device)
    hist = torch.empty(16 * 256, dtype=torch.int32, device=device)
    _native.check(lib.pbsm_pair_digits(out.data_ptr(), n, hist.data_ptr(), stream),
                  "pbsm_pair_digits")
    full = (hist.view(16, 256) == n).any(1).cpu().tolist()  # one bucket holds every key
    mask = sum(1 << d for d in range(16) if not full[d])
    if mask:
        tmp = torch.empty_like(out)
        scratch = torch.empty(int(lib.pbsm_sort_pairs_scratch_bytes(n)), dtype=torch.uint8,
                              device=device)
        _native.check(lib.pbsm_sort_pairs(out.data_ptr(), n, mask, tmp.data_ptr(),
                                          scratch.data_ptr(), stream), "pbsm_sort_pairs")
    return out


# ---------------------------------------------------------------- CUDA graphs
# The repeated-shape path as one graph per (inputs, shape, sizes): its
# enqueue sequence is fixed once the plan sizes are known (speculative sizes
# from the previous join of the shape), so it is captured once and replayed —
# the ~12 launches and their host work (~100 µs of Python + driver calls per
# join, the whole cost of a near-empty join) become one graph launch.
GRAPHS = os.environ.get("PBSM_GRAPHS", "1") != "0"
# tests: capture the header all_gather even on a one-rank group (the
# collective path of a multi-GPU run, exercised on one GPU)
GRAPH_EXCHANGE_ALWAYS = os.environ.get("PBSM_GRAPH_EXCHANGE_ALWAYS") == "1"
_graph_cache: dict = {}


class _Graphed:
    def __init__(self):
        self.graph = None
        self.hdr = None      # page-locked header the graph's last kernel writes
        self.pairs = None
        self.keep = []       # buffers the graph's kernels address
        self.gathered = None  # page-locked (world, HDR_WORDS + 5): every rank's header + caps
        self.world = 1
        # fast replay (_fast_replay): the inputs this graph reads (kept alive:
        # their ids key the lookup), their addresses, the header as int64
        # words, the speculative caps, the last result's pair view
        self.inputs = None
        self.ptrs = ()
        self.hdr_words = None
        self.cap_list = ()
        self.view = (-1, None)


HDR_WORDS = C.sizeof(_native.Header) // 8
_CAPS = ("list_r", "list_s", "nested", "other", "pairs", "nested_r", "nested_s")


def _guess_missed(h: dict, caps) -> bool:
    """Did a join sized from the speculative ``caps`` (list_r, list_s, nested
    chunks, other units, pairs) miss its true plan ``h``?"""
    return bool(h["list_r"] > caps[0] or h["list_s"] > caps[1] or h["chunks_nested"] > caps[2]
                or h["chunks_sorted"] + h["n_items"] > caps[3] or h["pairs"] > caps[4]
                or h["nested_r"] > caps[5] or h["nested_s"] > caps[6]
                or h["error"] & (_native.ERR_PAIR_OVERFLOW | _native.ERR_SCATTER_OVERFLOW))


def _header_row(row) -> dict:
    """An int64 row of HDR_WORDS header words → the header dict."""
    h = _native.Header.from_buffer_copy(bytes(memoryview(row[:HDR_WORDS].copy())))
    return h.as_dict()


def _graph_enqueue(lib, g: _Graphed, r: DeviceRects, s: DeviceRects, grid, guess,
                   nested_max: int, sweep_min: int, device, side_st) -> None:
    """The speculative path's launches (run_join, guess given), on the current
    stream and one side stream, nothing synchronous — captured into g.graph."""
    main_st = torch.cuda.current_stream(device)
    stream = main_st.cuda_stream
    kx, ky, row_lo, row_hi = grid
    ws = torch.empty(int(lib.pbsm_workspace_bytes(*grid)), dtype=torch.uint8, device=device)
    wsp = ws.data_ptr()
    list_r, list_s = guess["list_r"], guess["list_s"]
    same = SELF_ONCE and s is r  # a self-join: one count, one scatter, one list
    lists = [torch.empty((max(list_r, 1), 8), dtype=torch.int64, device=device)]
    lists.append(lists[0] if same else
                 torch.empty((max(list_s, 1), 8), dtype=torch.int64, device=device))
    cap, cn, rest = guess["pairs"], guess["nested"], guess["other"]
    lcap, mtile = guess["large"], guess["max_huge"]
    scratch = torch.empty(int(lib.pbsm_join_scratch_bytes(cn + rest, lcap)), dtype=torch.uint8,
                          device=device)
    g.pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=device)
    g.keep += [ws, lists, scratch]
    nest = (guess["nested_r"], guess["nested_s"])
    split = _split_ok(True, None, False, False, nest[0], nest[1], len(r), len(s),
                      guess["count"], False)
    split_bufs = []
    if split:
        split_bufs = [(torch.empty((max(nest[q], 1), 4), dtype=torch.int64, device=device),
                       max(nest[q], 1)) for q in range(1 if same else 2)]
        if same:
            split_bufs.append(split_bufs[0])
        g.keep.append(split_bufs)

    def fork():
        e = torch.cuda.Event()
        e.record(main_st)
        side_st.wait_event(e)

    def join():
        e = torch.cuda.Event()
        e.record(side_st)
        main_st.wait_event(e)

    _native.check(lib.pbsm_init(wsp, *grid, stream), "pbsm_init")
    if same:
        _native.check(lib.pbsm_count(_ptr(r.xl), _ptr(r.xu), _ptr(r.yl), _ptr(r.yu), len(r), 0,
                                     wsp, *grid, stream), "pbsm_count")
        cnt_r_v, cnt_s_v = _tile_count_views(ws, kx, ky, kx * (row_hi - row_lo))
        cnt_s_v.copy_(cnt_r_v, non_blocking=True)
    else:
        fork()
        for side, b in ((0, r), (1, s)):
            _native.check(lib.pbsm_count(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), len(b),
                                         side, wsp, *grid,
                                         side_st.cuda_stream if side else stream), "pbsm_count")
        join()
    _native.check(lib.pbsm_plan(wsp, *grid, nested_max, sweep_min, stream), "pbsm_plan")
    if not same:
        fork()
    for side, b, total in (((0, r, list_r),) if same else ((0, r, list_r), (1, s, list_s))):
        st_ = side_st.cuda_stream if side else stream
        if split:
            rec32, n32 = split_bufs[side]
            _native.check(lib.pbsm_scatter_split(_ptr(b.ids), _ptr(b.xl), _ptr(b.xu), _ptr(b.yl),
                                                 _ptr(b.yu), len(b), side, wsp, *grid,
                                                 lists[side].data_ptr(), total, rec32.data_ptr(),
                                                 n32, st_), "pbsm_scatter_split")
        else:
            _native.check(lib.pbsm_scatter(_ptr(b.ids), _ptr(b.xl), _ptr(b.xu), _ptr(b.yl),
                                           _ptr(b.yu), len(b), side, wsp, *grid,
                                           lists[side].data_ptr(), total, st_), "pbsm_scatter")
    if not same:
        join()
    if split:
        _emit_split(lib, wsp, grid, lists[0], list_r, lists[1], list_s, split_bufs, r, s, False,
                    None, (cn, rest, lcap, mtile), scratch, g.pairs, cap, stream, guess["count"])
    else:
        _native.check(lib.pbsm_join_emit_bounded(wsp, *grid, lists[0].data_ptr(), list_r,
                                                 lists[1].data_ptr(), list_s, cn, rest, lcap,
                                                 mtile, scratch.data_ptr(), g.pairs.data_ptr(),
                                                 cap, stream), "pbsm_join_emit_bounded")
    _native.check(lib.pbsm_publish_header(wsp, g.hdr.data_ptr(), stream), "pbsm_publish_header")
    if g.gathered is not None:
        # the join's one collective, from the device header (no host round
        # trip): every rank's header words + the caps its graph was sized
        # with, so every rank can tell whether ANY rank's sizes missed
        import torch.distributed as dist

        mine = torch.cat([ws[:8 * HDR_WORDS].view(torch.int64), g.caps])
        allv = torch.empty((g.world, HDR_WORDS + len(_CAPS)), dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(allv, mine)
        g.gathered.copy_(allv, non_blocking=True)
        g.keep += [mine, allv]


def _run_graphed(lib, r, s, kx, ky, row_lo, row_hi, key, guess, nested_max, sweep_min,
                 stream, exchange: bool = False) -> DeviceJoinResult | None:
    """run_join's repeated-shape path as a graph replay + one host sync.
    Returns None when the speculative sizes missed (the caller runs the
    exact path, which refreshes the sizes).  With ``exchange`` on several
    ranks the graph also all-gathers the headers; then a miss on any rank is
    handled here, identically on every rank: the ranks that missed re-run
    their join exactly, and all ranks exchange their counts eagerly."""
    device = r.device
    world, rank = 1, 0
    if exchange:
        import torch.distributed as dist

        if dist.is_initialized():
            world, rank = dist.get_world_size(), dist.get_rank()
    # (NCCL only: a gloo collective cannot be captured in a CUDA graph — the
    # eager exchange after the read serves those groups)
    gathered = exchange and dist.is_initialized() and dist.get_backend() == "nccl" and (
        world > 1 or GRAPH_EXCHANGE_ALWAYS)
    gkey = key + tuple(t.data_ptr() for t in r.columns() + s.columns()) + (
        tuple(sorted(guess.items())),)
    with _state_lock:
        g = _graph_cache.get(gkey)
    if g is None:
        with _state_lock:  # one graph per (device, stream): drop the previous shape's
            for k_ in [k_ for k_ in _graph_cache if k_[:2] == key[:2]]:
                del _graph_cache[k_]
        g = _Graphed()
        g.world = world
        g.hdr = torch.zeros(C.sizeof(_native.Header), dtype=torch.uint8, pin_memory=True)
        g.hdr_words = g.hdr.numpy().view(np.int64)
        g.cap_list = [int(guess[c]) for c in _CAPS]
        g.inputs = (r, s)
        g.ptrs = tuple(t.data_ptr() for t in r.columns() + s.columns())
        if gathered:
            g.gathered = torch.zeros((world, HDR_WORDS + len(_CAPS)), dtype=torch.int64,
                                     pin_memory=True)
            g.caps = torch.tensor([guess[c] for c in _CAPS], dtype=torch.int64).to(device)
        g.graph = torch.cuda.CUDAGraph()
        cap_stream = torch.cuda.Stream(device)
        side_st = torch.cuda.Stream(device)
        g.keep += [cap_stream, side_st]
        cap_stream.wait_stream(torch.cuda.current_stream(device))
        with torch.cuda.graph(g.graph, stream=cap_stream):
            _graph_enqueue(lib, g, r, s, (kx, ky, row_lo, row_hi), guess, nested_max, sweep_min,
                           device, side_st)
        torch.cuda.current_stream(device).wait_stream(cap_stream)
        with _state_lock:
            _graph_cache[gkey] = g
    g.graph.replay()
    torch.cuda.current_stream(device).synchronize()
    h2 = _native.Header.from_buffer_copy(C.string_at(g.hdr.data_ptr(), C.sizeof(_native.Header)))
    for bit, msg in _VALIDATION:
        if h2.error & bit:
            raise ValueError(msg)
    miss = _guess_missed(h2.as_dict(), [guess[c] for c in _CAPS])
    if miss:
        with _state_lock:
            _graph_cache.pop(gkey, None)
            _plan_cache.pop(key, None)
            _fast.pop(key[:2], None)
    if g.gathered is not None:
        rows = g.gathered.numpy().copy()
        misses = [_guess_missed(_header_row(rw), rw[HDR_WORDS:]) for rw in rows]
        if any(misses):  # (every rank sees the same rows: the same branch everywhere)
            if miss:
                res = run_join(r, s, kx, ky, row_lo=row_lo, row_hi=row_hi,
                               nested_max=nested_max, sweep_min=sweep_min)
            else:
                res = DeviceJoinResult(int(h2.pairs), g.pairs[:int(h2.pairs)],
                                       header=h2.as_dict())
            return _with_exchange(res, True)
        from .parallel import exchange_from_rows

        res = DeviceJoinResult(int(h2.pairs), g.pairs[:int(h2.pairs)], header=h2.as_dict())
        res.header["exchange"] = exchange_from_rows(
            [(int(rw[12]), int(rw[0]), int(rw[1])) for rw in rows], rank)
        return res
    if miss:
        return None
    bad = h2.error & ~_VALIDATION_BITS
    if bad:
        raise KernelError(f"device guard: {_native.describe_error(bad)} "
                          "(partition write overflow check, partition.py:229-233)")
    count = int(h2.pairs)
    if g.gathered is None:
        with _state_lock:  # the next join of these inputs replays without the lookups above
            _fast[key[:2]] = (_fast_key(r, s, key), g)
    return DeviceJoinResult(count, g.pairs[:count], header=h2.as_dict())


# Fast replay.  Between two joins of a repeated shape the GPU idles while the
# host works (tools/timeline.py: ~40 µs per join, a fifth of an 8-way strip's
# step): the result of join i is decoded, run_join returns, is called again,
# rebuilds its cache keys and launches the graph.  The last graphed join of a
# (device, stream) is therefore remembered under a key of object identities;
# a repeat skips every lookup and decodes the page-locked header straight
# from its int64 words.  Anything unusual — an error bit, a size miss, other
# options — drops the entry and takes the general path.
_fast: dict = {}
FAST_REPLAY = os.environ.get("PBSM_FAST_REPLAY", "1") != "0"
_HDR_NAMES = tuple(n for n, _ in _native.Header._fields_ if n not in ("error", "pad"))
_HDR_IX = {n: i for i, n in enumerate(_HDR_NAMES)}
_MISS_IX = tuple(_HDR_IX[n] for n in ("list_r", "list_s", "chunks_nested", "chunks_sorted",
                                      "n_items", "pairs", "nested_r", "nested_s"))


def _fast_key(r, s, key) -> tuple:
    return (id(r), id(s)) + key[2:]


def _fast_replay(r, s, kx, ky, row_lo, row_hi, nested_max, bin_bytes, sweep_min):
    device = r.device
    ent = _fast.get((str(device), _raw_stream(device)))
    if ent is None:
        return None
    fkey, g = ent
    if fkey != (id(r), id(s), kx, ky, row_lo, row_hi, len(r), len(s), s is r, nested_max,
                bin_bytes, sweep_min):
        return None
    if g.inputs[0] is not r or g.inputs[1] is not s or r.coords_ready is not None \
            or s.coords_ready is not None or r.ids_ready is not None \
            or g.ptrs != tuple(t.data_ptr() for t in r.columns() + s.columns()):
        return None
    g.graph.replay()
    torch.cuda.current_stream(device).synchronize()
    w = g.hdr_words.tolist()
    v = [w[i] for i in _MISS_IX]
    c = g.cap_list  # (_CAPS: list_r, list_s, nested, other, pairs, nested_r, nested_s)
    if (w[-1] & 0xffffffff) or v[0] > c[0] or v[1] > c[1] or v[2] > c[2] or v[3] + v[4] > c[3] \
            or v[5] > c[4] or v[6] > c[5] or v[7] > c[6]:
        with _state_lock:
            _fast.pop((str(device), _raw_stream(device)), None)
        return None  # (the general path replays, reads the same header and handles it)
    count = v[5]
    if g.view[0] != count:
        g.view = (count, g.pairs[:count])
    h = dict(zip(_HDR_NAMES, w))
    h["error"] = 0
    h["n_units"] = v[2] + v[3] + v[4]
    return DeviceJoinResult(count, g.view[1], header=h)


def _emit_split(lib, wsp, grid, rl, list_r, sl, list_s, split_bufs, r, s, late, plan, bounds,
                scratch, pairs, cap, stream, pairs_hint=None) -> None:
    """pbsm_join_emit_split over the compact nested entries: the exact yu
    columns by row, ids looked up at the emit (rows while the id columns are
    still in flight: mapped after the join)."""
    (r32, c32r), (s32, c32s) = split_bufs
    cn, rest, lcap, mtile = bounds
    # occupancy hint: few pairs per entry (the previous join of the shape)
    few = 1 if pairs_hint is not None and pairs_hint <= 0.25 * (c32r + c32s) else 0
    _native.check(lib.pbsm_join_emit_split(
        wsp, *grid, rl.data_ptr(), list_r, r32.data_ptr(), c32r, _ptr(r.yu),
        None if late else _ptr(r.ids), sl.data_ptr(), list_s, s32.data_ptr(), c32s, _ptr(s.yu),
        None if late else _ptr(s.ids), plan, cn, rest, lcap, mtile, scratch.data_ptr(),
        pairs.data_ptr(), cap, few, stream), "pbsm_join_emit_split")


def _map_ids(lib, pairs, count: int, r: DeviceRects, s: DeviceRects, cur, stream) -> None:
    """Row-index pairs → id pairs once the id columns have landed."""
    if count == 0:
        return
    _wait(r.ids_ready, cur)
    _wait(s.ids_ready, cur)
    _native.check(lib.pbsm_map_ids(pairs.data_ptr(), count, _ptr(r.ids), _ptr(s.ids), stream),
                  "pbsm_map_ids")


_d2h_streams: dict = {}
STAGED_MIN_PAIRS = 1 << 16


def staged_pairs_to_host(pairs: torch.Tensor, count: int, r: DeviceRects,
                         s: DeviceRects) -> np.ndarray:
    """Row-index pairs of a join whose id columns are still crossing PCIe →
    (r_id, s_id) pairs in page-locked host memory, group by group.

    The last-landing id column (S's; R's for a self-join) arrives in row
    chunks (to_device_pipelined).  pbsm_group_pairs splits the pairs by the
    chunk they need; as each chunk lands, its group is mapped to ids
    (pbsm_map_ids) and copied back on a device→host stream, so the copy back
    overlaps the rest of the upload (PCIe is full duplex) and only the last
    group's map and copy follow the last input byte.  The pair list is
    unordered (engine.py:61-62); groups are laid out in chunk order."""
    lib = _native.load()
    device = pairs.device
    stream = _raw_stream(device)
    cur = torch.cuda.current_stream(device)
    host = torch.empty((count, 2), dtype=torch.int64, pin_memory=True)
    if count == 0:
        return host.numpy()
    chunks = s.id_chunks
    if chunks is None or count < STAGED_MIN_PAIRS:
        _map_ids(lib, pairs, count, r, s, cur, stream)
        host.copy_(pairs[:count])
        return host.numpy()
    rows, evs = chunks
    g_n = len(evs)
    grouped = _buffer(device, "grouped", (count, 2), torch.int64, stream)
    cnt = _buffer(device, "group_counts", (2 * g_n,), torch.int64, stream)
    _native.check(lib.pbsm_group_pairs(pairs.data_ptr(), count, rows, g_n, int(s is r),
                                       grouped.data_ptr(), cnt.data_ptr(), stream),
                  "pbsm_group_pairs")
    sizes = torch.empty(g_n, dtype=torch.int64, pin_memory=True)
    sizes.copy_(cnt[:g_n], non_blocking=True)
    done = torch.cuda.Event()
    done.record(cur)
    done.synchronize()  # (the ids are still landing: the host has time)
    sizes = sizes.tolist()
    if sum(sizes) != count:
        raise KernelError(f"pbsm_group_pairs: groups hold {sum(sizes)} of {count} pairs")
    d2h = _d2h_streams.get(device.index)
    if d2h is None:
        d2h = _d2h_streams[device.index] = torch.cuda.Stream(device)
    if s is not r:
        _wait(r.ids_ready, cur)  # R's ids land before S's chunks
    off = 0
    for g, n_g in enumerate(sizes):
        cur.wait_event(evs[g])
        if n_g == 0:
            continue
        part = grouped[off:off + n_g]
        _native.check(lib.pbsm_map_ids(part.data_ptr(), n_g, _ptr(r.ids), _ptr(s.ids), stream),
                      "pbsm_map_ids")
        e = torch.cuda.Event()
        e.record(cur)
        d2h.wait_event(e)
        with torch.cuda.stream(d2h):
            host[off:off + n_g].copy_(part, non_blocking=True)
        off += n_g
    d2h.synchronize()
    cur.wait_stream(d2h)  # later work on the main stream may reuse the buffers
    return host.numpy()


def tile_counts(r, s, kx: int, ky: int, row_lo: int = 0, row_hi: int | None = None,
                device=None):
    """Per-tile assignment counts of both inputs (count_pass,
    partition.py:136-148; count_tiles, _kernels.pyx:34-58) as int64 numpy
    arrays of kx × (row_hi-row_lo) tiles, row-major.  ``r``/``s`` are host
    batches (RectBatch / 5-tuples) or DeviceRects; one pbsm_init + pbsm_count
    per input on the device, nothing else of the join runs.  Validation
    errors raise the reference's ValueError."""
    lib = _native.load()
    if row_hi is None:
        row_hi = ky
    if not isinstance(r, DeviceRects):
        dv = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        same = s is None or s is r
        r = to_device(r, dv)
        s = r if same else (s if isinstance(s, DeviceRects) else to_device(s, dv))
    elif s is None:
        s = r
    device = r.device
    stream = _raw_stream(device)
    ws = _workspace(lib, device, kx, ky, row_lo, row_hi, stream)
    wsp = ws.data_ptr()
    grid = (kx, ky, row_lo, row_hi)
    _native.check(lib.pbsm_init(wsp, *grid, stream), "pbsm_init")
    for side, b in ((0, r), (1, s)):
        if len(b):
            _native.check(lib.pbsm_count(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), len(b),
                                         side, wsp, *grid, stream), "pbsm_count")
    T = kx * (row_hi - row_lo)
    cr, cs = (v.to(torch.int64) for v in _tile_count_views(ws, kx, ky, T))
    out = (cr.cpu().numpy(), cs.cpu().numpy())
    _read_header(lib, ws, stream)  # validation bits → ValueError
    return out


def partition_columns(batch, kx: int, ky: int, device=None):
    """partition() on the device (partition.py:243-263): every rectangle of
    ``batch`` (RectBatch / 5-tuple) copied into each tile of the ``kx × ky``
    grid it overlaps, tile-major and in input order inside a tile (the
    reference's order for every writer count).  Returns host numpy arrays
    (offsets int64[kx*ky+1], ids, xl, xu, yl, yu) — PartitionedDataset's
    fields (partition.py:75-111).  RectBatch.validate's errors are the
    caller's (the reference validates in as_batch / join)."""
    lib = _native.load()
    dv = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    b = batch if isinstance(batch, DeviceRects) else to_device(batch, dv)
    n = len(b)
    stream = _raw_stream(b.device)
    scratch = torch.empty(int(lib.pbsm_partition_scratch_bytes(n, kx, ky)), dtype=torch.uint8,
                          device=b.device)
    total_d = torch.empty(1, dtype=torch.int64, device=b.device)
    _native.check(lib.pbsm_partition_count(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), n, kx,
                                           ky, scratch.data_ptr(), total_d.data_ptr(), stream),
                  "pbsm_partition_count")
    a = int(total_d.item())
    keys = torch.empty((max(a, 1), 2), dtype=torch.int64, device=b.device)
    tmp = torch.empty_like(keys)
    sort_scratch = torch.empty(int(lib.pbsm_sort_pairs_scratch_bytes(a)), dtype=torch.uint8,
                               device=b.device)
    out = [torch.empty(max(a, 1), dtype=torch.int64, device=b.device)] + [
        torch.empty(max(a, 1), dtype=torch.float64, device=b.device) for _ in range(4)]
    offsets = torch.empty(kx * ky + 1, dtype=torch.int64, device=b.device)
    _native.check(lib.pbsm_partition_write(
        _ptr(b.ids), _ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), n, kx, ky,
        scratch.data_ptr(), a, keys.data_ptr(), tmp.data_ptr(), sort_scratch.data_ptr(),
        *(t.data_ptr() for t in out), offsets.data_ptr(), stream), "pbsm_partition_write")
    return (offsets.cpu().numpy(),) + tuple(t[:a].cpu().numpy() for t in out)


def _align(v: int, a: int = 256) -> int:
    return (v + a - 1) // a * a


def _tile_count_views(ws: torch.Tensor, kx: int, ky: int, T: int):
    """(cnt_r, cnt_s) int32 views into the workspace (mirrors ws_layout in pbsm.cu)."""
    o = _align(C.sizeof(_native.Header))
    o = _align(o + 8 * (kx + 1))
    o = _align(o + 8 * (ky + 1))
    cr = ws[o:o + 4 * T].view(torch.int32)
    o = _align(o + 4 * T)
    cs = ws[o:o + 4 * T].view(torch.int32)
    return cr, cs
