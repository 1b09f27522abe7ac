"""Drop-in join API: ``join`` / ``epsilon_distance_join`` on the B200.

Same entry points, configuration object, report object and error behaviour
as the reference engine (/root/reference/pkg/src/sweepjoin/engine.py:35-70,
103-120, 312-353); the whole filter step runs in the sm_100a library
(``device.run_join``).  ``axis_policy``, ``threads``, ``phi``, ``k_buckets``
and ``backend`` are validated exactly like the reference and otherwise
ignored: the sweep axis and thread count never change the result set
(sweep.py:131-132), and there is one backend.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Literal, NamedTuple, Sequence

import numpy as np
import torch

from . import device as dev
from .errors import ConfigError, KernelError
from .geometry import Rect, RectBatch, as_batch
from .partition import MAX_DEVICE_K, PartitionedDataset, PartitionLayout

AxisPolicyName = Literal["x", "y", "adaptive", "auto"]

__all__ = ["JoinConfig", "JoinReport", "JoinTask", "SortTask", "build_task_queue",
           "epsilon_distance_join", "join", "join_device", "squares"]


@dataclass
class JoinConfig:
    """Parameters of one join (engine.py:35-52 in the reference).

    ``devices`` is new: the number of GPUs of a strip-sharded join (see
    ``parallel.py``); the single-process ``join`` uses the current device.
    """

    layout: PartitionLayout
    axis_policy: AxisPolicyName | None = None
    threads: int = 1
    sink_mode: Literal["count-only", "collect-pairs"] = "count-only"
    phi: int | None = None
    k_buckets: int | None = None
    backend: str | None = None
    devices: int = 1


class _Lazy:
    """Dataclass field whose value may be given as a zero-argument callable,
    evaluated once on first read (the field stays an ordinary constructor
    argument: ``JoinReport(..., task_sizes=array)`` works as in the reference)."""

    def __set_name__(self, owner, name):
        self.slot = "_lazy_" + name

    def __get__(self, obj, objtype=None):
        if obj is None:
            return None
        v = obj.__dict__.get(self.slot)
        if callable(v):
            v = v()
            obj.__dict__[self.slot] = v
        return v

    def __set__(self, obj, value):
        obj.__dict__[self.slot] = None if isinstance(value, _Lazy) else value


@dataclass
class JoinReport:
    """Result size, optional ``(n, 2)`` int64 (r_id, s_id) pairs and phase times.

    Field meanings follow engine.py:55-70.  ``sort_time`` is 0.0: the
    per-tile sort is fused into the join kernels and accounted in
    ``join_time``.  ``task_sizes`` (|R_T|+|S_T| of every join tile, largest
    first, build_task_queue engine.py:84-100) is computed on first read by a
    device count pass over the HOST inputs the report references — a report
    holds no device memory.
    """

    result_count: int
    pairs: np.ndarray | None
    partition_time: float
    sort_time: float
    join_time: float
    total_time: float
    task_sizes: np.ndarray | None = field(default=_Lazy(), repr=False)


class SortTask(NamedTuple):
    """One per-tile sort (engine.py:73-76); ``which`` 0 = first input, 1 = second."""

    which: int
    tile: int
    size: int


class JoinTask(NamedTuple):
    """One per-tile join (engine.py:79-81)."""

    tile: int
    size: int


def build_task_queue(partitioned_r: PartitionedDataset, partitioned_s: PartitionedDataset,
                     ) -> tuple[list[SortTask], list[JoinTask]]:
    """The reference's work lists, largest first (engine.py:84-100): one sort
    task per non-empty (tile, input), one join task per tile where both
    inputs are non-empty.  (The device join builds the same join set and its
    own CTA work units inside pbsm_plan; this is the host view of it.)"""
    cr, cs = partitioned_r.counts, partitioned_s.counts
    sort_tasks = [SortTask(0, int(t), int(cr[t])) for t in np.nonzero(cr)[0]]
    sort_tasks += [SortTask(1, int(t), int(cs[t])) for t in np.nonzero(cs)[0]]
    sort_tasks.sort(key=lambda task: -task.size)
    both = np.nonzero((cr > 0) & (cs > 0))[0]
    join_tasks = [JoinTask(int(t), int(cr[t] + cs[t])) for t in both]
    join_tasks.sort(key=lambda task: -task.size)
    return sort_tasks, join_tasks


def _resolve_policy(cfg: JoinConfig) -> str:
    """Config validation with the reference's messages (engine.py:103-120)."""
    if cfg.threads < 1:
        raise ConfigError("threads must be >= 1")
    if cfg.sink_mode not in ("count-only", "collect-pairs"):
        raise ConfigError(f"unknown sink mode {cfg.sink_mode!r}")
    if cfg.phi is not None and cfg.phi < 1:
        raise ConfigError("phi must be >= 1")
    if cfg.k_buckets is not None and cfg.k_buckets < 1:
        raise ConfigError("k_buckets must be >= 1")
    policy = cfg.axis_policy
    if policy is None:
        policy = "auto" if cfg.layout.kind == "1d" else "adaptive"
    if policy not in ("x", "y", "adaptive", "auto"):
        raise ConfigError(f"unknown axis policy {policy!r}")
    if policy == "auto" and cfg.layout.kind != "1d":
        raise ConfigError("axis policy 'auto' applies to 1D stripes only; "
                          "use 'adaptive' for grids")
    if cfg.backend not in (None, "cuda", "b200"):
        raise ValueError(f"unknown backend {cfg.backend!r}; available: ('cuda',)")
    if cfg.layout.k > MAX_DEVICE_K:
        raise ConfigError(f"k={cfg.layout.k} exceeds the device limit {MAX_DEVICE_K}")
    if cfg.devices < 1:
        raise ConfigError("devices must be >= 1")
    return policy


def _to_host(t: torch.Tensor) -> np.ndarray:
    """Device → host into page-locked memory (torch's caching host allocator):
    a fresh pageable buffer would page-fault on every 4 KiB of the copy.  The
    returned array keeps its pinned tensor alive."""
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)
    return host.numpy()


def _require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise KernelError("no CUDA device: the B200 join has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _task_sizes_fn(r: RectBatch, s: RectBatch, kx: int, ky: int, eps: float | None = None):
    """Lazy task_sizes: the report keeps references to the caller's host
    batches only; on first read their coordinates go back to the device for
    one count pass (pbsm_count; an ε-join's squares are built first) and the
    join tiles' sizes come back sorted."""
    def compute():
        if eps is not None:
            sr = squares(r, eps)
            cr, cs = dev.tile_counts(sr, sr if s is r else squares(s, eps), kx, ky)
        else:
            cr, cs = dev.tile_counts(r, s, kx, ky)
        both = (cr > 0) & (cs > 0)
        sizes = (cr + cs)[both]
        return -np.sort(-sizes, kind="stable")
    return compute


def join_device(r: dev.DeviceRects, s: dev.DeviceRects, cfg: JoinConfig,
                timing: bool = False) -> dev.DeviceJoinResult:
    """Device-resident join: inputs and the pair tensor stay in HBM."""
    _resolve_policy(cfg)
    kx, ky = cfg.layout.grid
    return dev.run_join(r, s, kx, ky, collect=cfg.sink_mode == "collect-pairs", timing=timing)


def _run(r: RectBatch, s: RectBatch, cfg: JoinConfig, t0: float,
         eps: float | None = None) -> JoinReport:
    collect_user = cfg.sink_mode == "collect-pairs"
    if len(r) == 0 or len(s) == 0:
        return JoinReport(0, np.empty((0, 2), dtype=np.int64) if collect_user else None,
                          0.0, 0.0, 0.0, time.perf_counter() - t0,
                          task_sizes=np.empty(0, dtype=np.int64))
    device = _require_cuda()
    kx, ky = cfg.layout.grid
    if eps is not None:
        # ε-join: only the point columns cross PCIe (the squares are built
        # in the kernels, the distance test runs inside the mini-joins)
        rd = dev.points_to_device(r, device)
        sd = rd if s is r else dev.points_to_device(s, device)
        res = dev.run_join(rd, sd, kx, ky, collect=collect_user, timing=True, eps=eps)
    else:
        # column copies on a side stream, coordinates first: the count passes
        # start while the ids are still in flight; the pairs come back as row
        # indices and go home group by group as the id chunks land
        # (dev.staged_pairs_to_host)
        rd, sd = dev.to_device_pipelined(r, s, device)
        res = dev.run_join(rd, sd, kx, ky, collect=collect_user, timing=True,
                           defer_map=dev.STAGED and collect_user)
    count, pairs = res.count, res.pairs
    out = None
    if collect_user:
        if res.rows_pending:
            out = dev.staged_pairs_to_host(pairs, count, rd, sd)
        else:
            out = _to_host(pairs) if count else np.empty((0, 2), dtype=np.int64)
    t = res.times
    return JoinReport(
        result_count=int(count), pairs=out,
        partition_time=t.get("partition", 0.0), sort_time=0.0,
        join_time=t.get("join", 0.0),
        total_time=time.perf_counter() - t0,
        task_sizes=_task_sizes_fn(r, s, kx, ky, eps))


def join(r: RectBatch | Sequence[Rect], s: RectBatch | Sequence[Rect],
         cfg: JoinConfig) -> JoinReport:
    """Every intersecting (r, s) pair of R × S exactly once (engine.py:312-323)."""
    r, s = as_batch(r), as_batch(s)
    _resolve_policy(cfg)
    if len(r) == 0 or len(s) == 0 or not torch.cuda.is_available():
        r.validate()
        s.validate()
    # otherwise RectBatch.validate runs on the device inside the count pass
    # (same checks, same ValueError messages and order: R before S); without
    # a device the host check keeps the reference's ValueError ahead of the
    # KernelError "no CUDA device"
    return _run(r, s, cfg, time.perf_counter())


def squares(batch: RectBatch, eps: float, ids: np.ndarray | None = None) -> RectBatch:
    """Side-``eps`` squares around the lower corners, clipped to [0, 1].

    Exactly the numpy arithmetic of engine.py:342-350 (half = eps / 2.0).
    ``ids`` defaults to row indices, as the reference uses for refinement.
    """
    half = eps / 2.0
    return RectBatch(
        np.arange(len(batch), dtype=np.int64) if ids is None else ids,
        np.clip(batch.xl - half, 0.0, 1.0), np.clip(batch.xl + half, 0.0, 1.0),
        np.clip(batch.yl - half, 0.0, 1.0), np.clip(batch.yl + half, 0.0, 1.0))


def epsilon_distance_join(p: RectBatch | Sequence[Rect], q: RectBatch | Sequence[Rect],
                          eps: float, cfg: JoinConfig) -> JoinReport:
    """Point pairs within distance ``eps`` exactly once (engine.py:326-353).

    The points are the lower corners of ``p`` / ``q`` (engine.py:333-334).
    Candidates are the pairs whose side-``eps`` squares intersect (squares
    built in the kernels with the reference's arithmetic, engine.py:342-350);
    the distance test ``dx*dx + dy*dy <= eps*eps`` (numpy rounding, no FMA
    contraction, engine.py:201-206) runs inside the mini-joins, in the count
    pass and the emit alike, so only refined pairs are ever written.
    """
    if not eps > 0.0:
        raise ConfigError(f"epsilon must be positive, got {eps!r}")
    p, q = as_batch(p), as_batch(q)
    _resolve_policy(cfg)
    p.validate()
    q.validate()
    return _run(p, q, cfg, time.perf_counter(), eps=float(eps))
