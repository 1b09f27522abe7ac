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
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import KernelError

__all__ = ["DeviceRects", "DeviceJoinResult", "run_join", "to_device"]


@dataclass
class DeviceRects:
    """One input on the GPU in the reference's SoA column order."""

    ids: torch.Tensor   # int64 [n]
    xl: torch.Tensor    # float64 [n]
    xu: torch.Tensor
    yl: torch.Tensor
    yu: torch.Tensor

    def __len__(self) -> int:
        return int(self.ids.shape[0])

    @property
    def device(self) -> torch.device:
        return self.ids.device

    def columns(self):
        return self.ids, self.xl, self.xu, self.yl, self.yu


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


@dataclass
class DeviceJoinResult:
    count: int
    pairs: torch.Tensor | None          # int64 [P, 2] (r_id, s_id) on the device
    header: dict = field(default_factory=dict)
    times: dict = field(default_factory=dict)  # seconds per phase (CUDA events)
    tile_counts: tuple | None = None      # (cnt_r, cnt_s) device views when kept


_ws_cache: dict = {}


def _workspace(lib, device, kx, ky, row_lo, row_hi) -> torch.Tensor:
    key = (str(device), kx, ky, row_lo, row_hi)
    ws = _ws_cache.get(key)
    if ws is None:
        nbytes = lib.pbsm_workspace_bytes(kx, ky, row_lo, row_hi)
        if nbytes < 0:
            raise KernelError(f"invalid grid {kx}x{ky} rows [{row_lo},{row_hi})")
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device=device)
        _ws_cache.clear()  # keep one grid workspace alive at a time
        _ws_cache[key] = ws
    return ws


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None or t.numel() == 0 else t.data_ptr()


def _read_header(lib, ws, stream) -> _native.Header:
    h = _native.Header()
    _native.check(lib.pbsm_read_header(ws.data_ptr(), C.byref(h), stream), "pbsm_read_header")
    if h.error:
        raise KernelError(f"device guard: {_native.describe_error(h.error)} "
                          "(partition write overflow check, partition.py:229-233)")
    return h


def run_join(r: DeviceRects, s: DeviceRects, kx: int, ky: int, *, collect: bool = True,
             row_lo: int = 0, row_hi: int | None = None, timing: bool = False,
             keep_counts: bool = False) -> DeviceJoinResult:
    """Join two device-resident inputs over a ``kx × ky`` grid (rows [row_lo, row_hi))."""
    lib = _native.load()
    if row_hi is None:
        row_hi = ky
    device = r.device
    if len(r) == 0 or len(s) == 0:
        empty = torch.empty((0, 2), dtype=torch.int64, device=device) if collect else None
        return DeviceJoinResult(0, empty)
    stream = torch.cuda.current_stream(device).cuda_stream
    ws = _workspace(lib, device, kx, ky, row_lo, row_hi)
    wsp = ws.data_ptr()
    grid = (kx, ky, row_lo, row_hi)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timing else None
    if ev:
        ev[0].record()

    _native.check(lib.pbsm_init(wsp, *grid, stream), "pbsm_init")
    for side, b in ((0, r), (1, s)):
        _native.check(lib.pbsm_count(_ptr(b.xl), _ptr(b.xu), _ptr(b.yl), _ptr(b.yu), len(b),
                                     side, wsp, *grid, stream), "pbsm_count")
    _native.check(lib.pbsm_plan(wsp, *grid, stream), "pbsm_plan")
    h = _read_header(lib, ws, stream)

    lists = []
    for side, b, total in ((0, r, h.a_r), (1, s, h.a_s)):
        ent = torch.empty((max(total, 1), 4), dtype=torch.float64, device=device)
        eid = torch.empty(max(total, 1), dtype=torch.int64, device=device)
        _native.check(lib.pbsm_scatter(_ptr(b.ids), _ptr(b.xl), _ptr(b.xu), _ptr(b.yl),
                                       _ptr(b.yu), len(b), side, wsp, *grid, ent.data_ptr(),
                                       eid.data_ptr(), total, stream), "pbsm_scatter")
        lists.append((ent, eid))
    if ev:
        ev[1].record()

    n_chunks, n_items = h.n_chunks, h.n_items
    scratch = torch.empty(int(lib.pbsm_join_scratch_bytes(n_chunks, n_items)),
                          dtype=torch.uint8, device=device)
    (rl, rid), (sl, sid) = lists
    _native.check(lib.pbsm_join_count(wsp, *grid, rl.data_ptr(), sl.data_ptr(), n_chunks,
                                      n_items, scratch.data_ptr(), stream), "pbsm_join_count")
    h2 = _read_header(lib, ws, stream)
    if ev:
        ev[2].record()
    count = int(h2.pairs)
    pairs = None
    if collect:
        pairs = torch.empty((max(count, 1), 2), dtype=torch.int64, device=device)
        _native.check(lib.pbsm_join_emit(wsp, *grid, rl.data_ptr(), rid.data_ptr(),
                                         sl.data_ptr(), sid.data_ptr(), n_chunks, n_items,
                                         scratch.data_ptr(), pairs.data_ptr(), 0, count,
                                         stream), "pbsm_join_emit")
        h2 = _read_header(lib, ws, stream)
        pairs = pairs[:count]
    if ev:
        ev[3].record()
        ev[3].synchronize()
    res = DeviceJoinResult(count, pairs, header=h2.as_dict())
    if ev:
        res.times = {
            "partition": ev[0].elapsed_time(ev[1]) / 1e3,
            "join_count": ev[1].elapsed_time(ev[2]) / 1e3,
            "emit": ev[2].elapsed_time(ev[3]) / 1e3,
            "total": ev[0].elapsed_time(ev[3]) / 1e3,
        }
    if keep_counts:
        T = kx * (row_hi - row_lo)
        # the workspace is reused by the next join: hand out copies
        res.tile_counts = tuple(v.clone() for v in _tile_count_views(ws, kx, ky, T))
    return res


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
