"""GPU parity of the unit pipeline (units.cuh) against the reference fixtures,
and against the tile-list pipeline on the same inputs."""

import numpy as np
import pytest
import torch

import oracle
import paper_1908_11740_b200 as pb
from paper_1908_11740_b200 import device as dev
from paper_1908_11740_b200 import parallel
from paper_1908_11740_b200.synth import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _units_header(res):
    assert res.header.get("pipeline") == "units", res.header
    return res.header


def test_unit_pipeline_reference_instances(golden):
    """All 48 reference instances (mixed extents, boundary-snapped, points,
    1D and 2D layouts, self-joins) through the unit pipeline, forced."""
    g = golden["instances"]
    for row in g["cases"]:
        tag, kind, k, axis, self_join, count = str(row).split(",")
        k, axis, count = int(k), int(axis), int(count)
        r = tuple(g[f"{tag}_r_{c}"] for c in ("ids", "xl", "xu", "yl", "yu"))
        s = r if self_join == "1" else tuple(g[f"{tag}_s_{c}"] for c in
                                             ("ids", "xl", "xu", "yl", "yu"))
        kx, ky = pb.PartitionLayout(kind, k, pb.Axis(axis)).grid
        if len(r[0]) == 0 or len(s[0]) == 0:
            continue
        R = dev.to_device(r)
        S = R if s is r else dev.to_device(s)
        res = dev.run_join(R, S, kx, ky, pipeline="units")
        _units_header(res)
        assert res.count == count, tag
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), g[f"{tag}_pairs"]), tag


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_unit_pipeline_configs(golden, cfg):
    g = golden["configs"]
    r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
    R = dev.to_device(r)
    S = R if s is r else dev.to_device(s)
    for _ in range(3):  # synchronous sizes, then speculative ones
        res = dev.run_join(R, S, k, k, pipeline="units")
        h = _units_header(res)
        assert res.count == int(g[f"cfg{cfg}_count"])
        assert (h["a_r"], h["a_s"]) == (int(g[f"cfg{cfg}_a_r"]), int(g[f"cfg{cfg}_a_s"]))
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), g[f"cfg{cfg}_pairs"])
    cnt = dev.run_join(R, S, k, k, pipeline="units", collect=False)
    assert cnt.count == int(g[f"cfg{cfg}_count"]) and cnt.pairs is None


@pytest.mark.parametrize("target", [2, 64, 1 << 20])
def test_unit_sizes_do_not_change_the_result(golden, monkeypatch, target):
    """Units of ~2 records (every cell its own unit), 64, or whole rows: the
    same pair list; the strips of a 3-way plan reassemble it."""
    monkeypatch.setattr(dev, "UNIT_TARGET", target)
    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    R, S = dev.to_device(r), dev.to_device(s)
    res = dev.run_join(R, S, k, k, pipeline="units")
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), g["cfg2_pairs"])
    parts = []
    for lo, hi in zip(*(lambda c: (c[:-1], c[1:]))(parallel.plan_strips(r, s, k, 3))):
        rs, ss_ = parallel.strip_inputs(r, k, lo, hi), parallel.strip_inputs(s, k, lo, hi)
        sres = dev.run_join(dev.to_device(rs), dev.to_device(ss_), k, k, row_lo=lo, row_hi=hi,
                            pipeline="units")
        parts.append(sres.pairs.cpu().numpy())
    assert np.array_equal(oracle.sorted_pairs(np.concatenate(parts)), g["cfg2_pairs"])


def test_unit_pipeline_large_tiles_and_dense_cells():
    """Few coarse tiles: most tiles exceed LMAX and go to the deferred
    large-tile kernel (k_ularge), including many work items per tile."""
    r, s, k = make_config(1, 0.5)
    for kk in (1, 2, 5, 16):
        want = oracle.sorted_pairs(oracle.join(r, s, "2d", kk)["pairs"])
        res = dev.run_join(dev.to_device(r), dev.to_device(s), kk, kk, pipeline="units")
        h = _units_header(res)
        assert h["n_def_tiles"] > 0, kk
        assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), want), kk


def test_unit_pipeline_speculative_mismatch(golden):
    """Same shape, different data: the cached sizes are too small, the device
    flags it, the join re-runs with the exact plan (bit-exact)."""
    g = golden["configs"]
    r, s, k = make_config(2, float(g["cfg2_scale"]))
    R, S = dev.to_device(r), dev.to_device(s)
    for _ in range(2):
        dev.run_join(R, S, k, k, pipeline="units")
    s2 = list(s)
    s2[2] = np.clip(s[2] * 1.0 + 0.02, 0.0, 1.0)
    s2[4] = np.clip(s[4] + 0.02, 0.0, 1.0)
    s2 = tuple(s2)
    got = dev.run_join(R, dev.to_device(s2), k, k, pipeline="units")
    want = oracle.sorted_pairs(oracle.join(r, s2, "2d", k)["pairs"])
    assert np.array_equal(oracle.sorted_pairs(got.pairs.cpu().numpy()), want)
    res = dev.run_join(R, S, k, k, pipeline="units")
    assert np.array_equal(oracle.sorted_pairs(res.pairs.cpu().numpy()), g["cfg2_pairs"])


def test_unit_pipeline_validation_errors():
    r, s, k = make_config(1, 0.05)
    bad = tuple(a.copy() for a in r)
    bad[1][3] = bad[2][3] + 0.1
    with pytest.raises(ValueError, match="inverted"):
        dev.run_join(dev.to_device(bad), dev.to_device(s), k, k, pipeline="units")
    bad = tuple(a.copy() for a in s)
    bad[4][7] = 1.5
    with pytest.raises(ValueError, match="outside"):
        dev.run_join(dev.to_device(r), dev.to_device(bad), k, k, pipeline="units")
