"""Host-side API, validation and C-ABI export checks (no GPU needed)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1908_11740_b200 as pb
from paper_1908_11740_b200 import _native
from paper_1908_11740_b200.geometry import axis_tile_index

ROOT = Path(__file__).resolve().parents[1]


def _cfg(kind="2d", k=4, **kw):
    return pb.JoinConfig(pb.PartitionLayout(kind, k), **kw)


def test_library_exports_every_header_symbol():
    lib = _native.load()
    header = (ROOT / "include" / "pbsm.h").read_text()
    names = set(re.findall(r"^\w[\w\s\*]*?\b(pbsm_\w+)\(", header, re.M))
    assert names, "no declarations parsed"
    assert names == set(_native.EXPORTED)
    for name in names:
        assert hasattr(lib, name), name
    assert lib.pbsm_abi_version() == _native.ABI_VERSION


def test_workspace_sizing_and_argument_errors():
    lib = _native.load()
    assert lib.pbsm_workspace_bytes(100, 100, 0, 100) > 4 * 100 * 100 * 6
    assert lib.pbsm_workspace_bytes(0, 100, 0, 100) < 0
    assert lib.pbsm_workspace_bytes(10, 10, 5, 5) < 0
    assert lib.pbsm_init(None, 4, 4, 0, 4, None) < 0
    assert lib.pbsm_join_scratch_bytes(-1, 0) < 0
    assert lib.pbsm_join_scratch_bytes(0, -1) < 0
    assert lib.pbsm_join_scratch_bytes(0, 0) > 0
    assert lib.pbsm_join_scratch_bytes(10, 1000) > lib.pbsm_join_scratch_bytes(10, 0)


@pytest.mark.parametrize("kw,exc", [
    (dict(threads=0), pb.ConfigError),
    (dict(sink_mode="bogus"), pb.ConfigError),
    (dict(axis_policy="diagonal"), pb.ConfigError),
    (dict(axis_policy="auto"), pb.ConfigError),
    (dict(phi=0), pb.ConfigError),
    (dict(k_buckets=0), pb.ConfigError),
])
def test_config_errors_match_reference(kw, exc):
    with pytest.raises(exc):
        pb.join([], [], _cfg(**kw))


def test_invalid_inputs_rejected():
    bad = pb.RectBatch([1], [0.5], [1.5], [0.0], [0.5])
    with pytest.raises(ValueError):
        pb.join(bad, bad, _cfg())
    inv = pb.RectBatch([1], [0.6], [0.5], [0.0], [0.5])
    with pytest.raises(ValueError):
        pb.join(inv, inv, _cfg())
    with pytest.raises(ValueError):
        pb.RectBatch([1, 2], [0.1], [0.2], [0.1], [0.2])
    with pytest.raises(pb.ConfigError):
        pb.epsilon_distance_join([], [], 0.0, _cfg())


def test_empty_inputs_need_no_device():
    rep = pb.join(pb.RectBatch.empty(), pb.RectBatch.empty(), _cfg(sink_mode="collect-pairs"))
    assert rep.result_count == 0 and rep.pairs.shape == (0, 2)
    one = pb.RectBatch.from_rects([pb.Rect(0, 0, 1, 0, 1)])
    assert pb.join(one, pb.RectBatch.empty(), _cfg()).result_count == 0


def test_layout_grid_mapping():
    assert pb.PartitionLayout("2d", 7).grid == (7, 7)
    assert pb.PartitionLayout("1d", 9).grid == (9, 1)
    assert pb.PartitionLayout("1d", 9, pb.Axis.Y).grid == (1, 9)
    lay = pb.PartitionLayout("2d", 4)
    assert pb.tiles_overlapping(pb.Rect(0, 0.25, 0.5, 0.0, 0.1), lay) == [1, 2]
    with pytest.raises(ValueError):
        pb.PartitionLayout("3d", 2)
    with pytest.raises(ValueError):
        pb.PartitionLayout("2d", 0)


def test_host_tile_index_matches_golden(golden):
    g = golden["tile_of"]
    sel = slice(0, None, 7)
    got = [axis_tile_index(float(p), int(k)) for p, k in zip(g["p"][sel], g["k"][sel])]
    assert np.array_equal(np.array(got), g["tile"][sel])


def test_no_cpu_fallback_without_cuda(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    r = pb.RectBatch.from_rects([pb.Rect(0, 0.1, 0.2, 0.1, 0.2)])
    with pytest.raises(pb.KernelError):
        pb.join(r, r, _cfg())
