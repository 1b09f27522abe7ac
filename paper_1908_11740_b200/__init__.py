"""B200-native PBSM spatial-join filter step (arXiv 1908.11740).

Drop-in for the reference ``sweepjoin`` join path: ``join(R, S,
JoinConfig(PartitionLayout("2d", K), sink_mode="collect-pairs"))`` returns the
same ``result_count`` and the same (r_id, s_id) pair set, computed by
hand-written sm_100a CUDA kernels (``csrc/pbsm.cu``) behind the C ABI in
``include/pbsm.h``.  There is no CPU fallback.
"""

from .engine import (
    JoinConfig,
    JoinReport,
    JoinTask,
    SortTask,
    build_task_queue,
    epsilon_distance_join,
    join,
    join_device,
    squares,
)
from .errors import (
    ConfigError,
    DatasetError,
    InvalidHistogramError,
    InvalidStatisticsError,
    KernelError,
    NormalizationError,
    SweepJoinError,
)
from .geometry import (
    Axis,
    Rect,
    RectBatch,
    TileExtent,
    as_batch,
    axis_tile_index,
    duplicate_test_1d,
    duplicate_test_2d,
    intersects,
    tile_boundary,
)
from .partition import (
    DEFAULT_K_MAX,
    PartitionedDataset,
    PartitionLayout,
    count_pass,
    partition,
    recommend_k,
    tiles_overlapping,
    write_pass,
)

__version__ = "0.1.0"


def available_backends() -> tuple[str, ...]:
    """The reference's backend registry (backends.py:25-26) has one entry here."""
    return ("cuda",)


def default_backend() -> str:
    return "cuda"
