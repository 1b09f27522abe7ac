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
from typing import Literal

import numpy as np

from .errors import InvalidStatisticsError
from .geometry import Axis, Rect, TileExtent, axis_tile_index, tile_boundary

DEFAULT_K_MAX = 20000
MAX_DEVICE_K = 65535

PartitionKind = Literal["1d", "2d"]

__all__ = ["DEFAULT_K_MAX", "PartitionLayout", "recommend_k", "tiles_overlapping"]


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
