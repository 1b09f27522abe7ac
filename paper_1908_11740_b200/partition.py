"""Partition layouts of the unit square (host-side description).

``PartitionLayout`` keeps the reference's constructor, validation and flat
tile numbering (``row * k + col``; /root/reference/pkg/src/sweepjoin/
partition.py:27-72).  On the device every layout is a ``kx × ky`` grid:

* ``"2d"`` K×K grid → ``kx = ky = K``;
* ``"1d"`` K stripes split along x → ``kx = K, ky = 1`` (flat tile = column);
* ``"1d"`` K stripes split along y → ``kx = 1, ky = K`` (flat tile = row).

so the same CUDA kernels serve grids and stripes, with the same flat tile ids
the reference uses (``_kernels.pyx:91``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Literal, Sequence

import numpy as np

from .errors import ConfigError, InvalidStatisticsError
from .geometry import Axis, Rect, RectBatch, TileExtent, as_batch, axis_tile_index, tile_boundary

DEFAULT_K_MAX = 20000
MAX_DEVICE_K = 65535

PartitionKind = Literal["1d", "2d"]

__all__ = ["DEFAULT_K_MAX", "PartitionLayout", "PartitionedDataset", "compute_segment_offsets",
           "count_pass", "partition", "recommend_k", "split_slices", "tiles_overlapping",
           "write_pass"]


@dataclass(frozen=True)
class PartitionLayout:
    """K stripes (``"1d"``) or a K×K grid (``"2d"``) over [0, 1]²."""

    kind: PartitionKind
    k: int
    partition_axis: Axis = Axis.X  # stripes only

    def __post_init__(self) -> None:
        if self.kind not in ("1d", "2d"):
            raise ValueError(f"unknown partition kind {self.kind!r}")
        if self.k < 1:
            raise ValueError("k must be >= 1")

    @property
    def n_tiles(self) -> int:
        return self.k * self.k if self.kind == "2d" else self.k

    @property
    def kind_code(self) -> int:
        return 1 if self.kind == "2d" else 0

    @property
    def axis_code(self) -> int:
        return int(self.partition_axis)

    @property
    def grid(self) -> tuple[int, int]:
        """(kx, ky) of the equivalent device grid."""
        if self.kind == "2d":
            return self.k, self.k
        return (self.k, 1) if self.partition_axis is Axis.X else (1, self.k)

    def tile_extent(self, t: int) -> TileExtent:
        if not 0 <= t < self.n_tiles:
            raise IndexError(f"tile {t} out of range for {self.n_tiles} tiles")
        k = self.k
        if self.kind == "1d":
            lo, hi = tile_boundary(t, k), tile_boundary(t + 1, k)
            if self.partition_axis is Axis.X:
                return TileExtent(lo, hi, 0.0, 1.0, row=t)
            return TileExtent(0.0, 1.0, lo, hi, row=t)
        row, col = divmod(t, k)
        return TileExtent(tile_boundary(col, k), tile_boundary(col + 1, k),
                          tile_boundary(row, k), tile_boundary(row + 1, k), row=row, col=col)

    def tile_extents(self) -> list[TileExtent]:
        return [self.tile_extent(t) for t in range(self.n_tiles)]


def tiles_overlapping(r: Rect, layout: PartitionLayout) -> list[int]:
    """Ascending flat ids of the tiles a closed rectangle is assigned to."""
    kx, ky = layout.grid
    c0, c1 = axis_tile_index(r.xl, kx), axis_tile_index(r.xu, kx)
    r0, r1 = axis_tile_index(r.yl, ky), axis_tile_index(r.yu, ky)
    return [row * kx + col for row in range(r0, r1 + 1) for col in range(c0, c1 + 1)]


def recommend_k(avg_extent_split_axis: float, kind: PartitionKind = "1d",
                k_max: int = DEFAULT_K_MAX) -> int:
    """Division count with tiles about ten average extents wide (partition.py:266-276)."""
    if not avg_extent_split_axis > 0.0:
        raise InvalidStatisticsError(
            f"average extent must be positive, got {avg_extent_split_axis!r}")
    return int(np.clip(round(1.0 / (10.0 * avg_extent_split_axis)), 1, k_max))


# ---------------------------------------------------------------- public partitioning
# The reference's two-pass partitioning API (partition.py:75-263), on the
# device: the count pass is pbsm_count (the join's k_count), the write pass
# pbsm_partition_write (assignment keys, stable radix sort, gather).  The
# reference's writers m and executor only choose how the CPU work is split;
# the buffers they produce are identical for every m (criterion 9,
# tests/test_acceptance.py:291-313), and so are these.

@dataclass
class PartitionedDataset:
    """Per-tile contiguous rectangle buffers of one input (partition.py:75-111):
    tile ``t`` owns rows [offsets[t], offsets[t+1]) of the coordinate arrays.
    ``hist_x`` / ``hist_y`` (the adaptive axis model's sampled histograms) are
    always None here: that model is out of scope (result-invariant)."""

    layout: PartitionLayout
    offsets: np.ndarray
    ids: np.ndarray
    xl: np.ndarray
    xu: np.ndarray
    yl: np.ndarray
    yu: np.ndarray
    source_count: int
    hist_x: np.ndarray | None = None
    hist_y: np.ndarray | None = None

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.offsets)

    @property
    def total_assigned(self) -> int:
        return int(self.offsets[-1])

    def tile_bounds(self, t: int) -> tuple[int, int]:
        return int(self.offsets[t]), int(self.offsets[t + 1])

    def tile_batch(self, t: int) -> RectBatch:
        lo, hi = self.tile_bounds(t)
        return RectBatch(self.ids[lo:hi], self.xl[lo:hi], self.xu[lo:hi],
                         self.yl[lo:hi], self.yu[lo:hi])


def split_slices(n: int, m: int) -> list[tuple[int, int]]:
    """range(n) in m near-equal contiguous [start, stop) slices (partition.py:130-133)."""
    bounds = np.linspace(0, n, m + 1).astype(np.int64)
    return [(int(bounds[i]), int(bounds[i + 1])) for i in range(m)]


def compute_segment_offsets(per_slice_counts: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(m, n_tiles) counts → (CSR tile offsets, each writer's start per tile)
    (partition.py:151-164)."""
    per_slice_counts = np.atleast_2d(np.asarray(per_slice_counts, dtype=np.int64))
    totals = per_slice_counts.sum(axis=0)
    tile_offsets = np.zeros(len(totals) + 1, dtype=np.int64)
    np.cumsum(totals, out=tile_offsets[1:])
    within = np.zeros_like(per_slice_counts)
    np.cumsum(per_slice_counts[:-1], axis=0, out=within[1:])
    return tile_offsets, within + tile_offsets[:-1]


def _check_hist(hist) -> None:
    if hist is not None:
        raise ConfigError("per-tile axis histograms belong to the adaptive axis model, "
                          "which this build does not implement (result-invariant)")


def count_pass(rects: RectBatch | Sequence[Rect], layout: PartitionLayout,
               start: int = 0, stop: int | None = None, kernels=None) -> np.ndarray:
    """Per-tile assignment counts of rows [start, stop) (partition.py:136-148),
    by the device count pass (pbsm_count).  ``kernels`` is accepted for
    signature compatibility; there is one backend."""
    from . import device as dev

    batch = as_batch(rects)
    if stop is None:
        stop = len(batch)
    kx, ky = layout.grid
    if stop <= start:
        return np.zeros(layout.n_tiles, dtype=np.int64)
    sl = tuple(np.ascontiguousarray(a[start:stop])
               for a in (batch.ids, batch.xl, batch.xu, batch.yl, batch.yu))
    return dev.tile_counts(sl, sl, kx, ky)[0]


def _device_dataset(batch: RectBatch, layout: PartitionLayout) -> PartitionedDataset:
    from . import device as dev

    kx, ky = layout.grid
    offsets, ids, xl, xu, yl, yu = dev.partition_columns(
        (batch.ids, batch.xl, batch.xu, batch.yl, batch.yu), kx, ky)
    return PartitionedDataset(layout, offsets, ids, xl, xu, yl, yu, source_count=len(batch))


def write_pass(rects: RectBatch | Sequence[Rect], layout: PartitionLayout,
               counts: np.ndarray, segment_offsets: np.ndarray,
               executor=None, kernels=None, hist=None) -> PartitionedDataset:
    """Fill the per-tile buffers (partition.py:176-240) on the device.  The
    reference's guard (:229-233) is kept: writer i (input slice i of m) must
    end exactly at writer i+1's start, the last at the tile's end, or
    RuntimeError — checked against the device count of each slice."""
    _check_hist(hist)
    batch = as_batch(rects)
    seg = np.atleast_2d(np.asarray(segment_offsets, dtype=np.int64))
    m = seg.shape[0]
    tile_offsets = np.zeros(layout.n_tiles + 1, dtype=np.int64)
    np.cumsum(np.asarray(counts, dtype=np.int64), out=tile_offsets[1:])
    final = np.vstack([seg[i] + count_pass(batch, layout, a, b)
                       for i, (a, b) in enumerate(split_slices(len(batch), m))])
    expected = np.vstack([seg[1:], tile_offsets[1:].reshape(1, -1)])
    if not np.array_equal(final, expected):
        raise RuntimeError("partition write overflow: count and write passes disagree")
    return _device_dataset(batch, layout)


def partition(rects: RectBatch | Sequence[Rect], layout: PartitionLayout,
              m: int = 1, executor=None, kernels=None, hist=None) -> PartitionedDataset:
    """Two-pass partitioning (partition.py:243-263): count, offsets, write —
    one device pass each; the result is the reference's for every ``m``."""
    _check_hist(hist)
    return _device_dataset(as_batch(rects), layout)
