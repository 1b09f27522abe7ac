"""Pin the CPU oracle against the reference's own outputs (tests/golden).

CPU-only: these tests validate the checker that the GPU parity tests rely on.
"""

import numpy as np
import pytest

import oracle
from paper_1908_11740_b200.synth import CONFIGS, make_config


def _case_list(golden):
    for row in golden["instances"]["cases"]:
        tag, kind, k, axis, self_join, count = str(row).split(",")
        yield tag, kind, int(k), int(axis), bool(int(self_join)), int(count)


def _side(g, tag, side):
    return tuple(g[f"{tag}_{side}_{c}"] for c in ("ids", "xl", "xu", "yl", "yu"))


def test_tile_of_known_answers(golden):
    g = golden["tile_of"]
    p, k, t = g["p"], g["k"], g["tile"]
    got = np.array([oracle.tile_of(float(a), int(b)) for a, b in zip(p, k)])
    assert np.array_equal(got, t)


@pytest.mark.parametrize("sweep_axis", [0, 1])
def test_oracle_matches_reference_instances(golden, sweep_axis):
    g = golden["instances"]
    n = 0
    for tag, kind, k, axis, self_join, count in _case_list(golden):
        r = _side(g, tag, "r")
        s = r if self_join else _side(g, tag, "s")
        res = oracle.join(r, s, kind, k, part_axis=axis, sweep_axis=sweep_axis, threads=2)
        assert res["count"] == count, tag
        assert np.array_equal(oracle.sorted_pairs(res["pairs"]), g[f"{tag}_pairs"]), tag
        n += 1
    assert n >= 40


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_oracle_matches_reference_configs(golden, cfg):
    g = golden["configs"]
    r, s, k = make_config(cfg, float(g[f"cfg{cfg}_scale"]))
    res = oracle.join(r, s, "2d", k, threads=4)
    assert res["count"] == int(g[f"cfg{cfg}_count"])
    assert res["a_r"] == int(g[f"cfg{cfg}_a_r"])
    assert res["a_s"] == int(g[f"cfg{cfg}_a_s"])
    assert np.array_equal(oracle.sorted_pairs(res["pairs"]), g[f"cfg{cfg}_pairs"])


def test_oracle_tile_counts_cfg1(golden):
    g = golden["configs"]
    r, s, k = make_config(1)
    assert np.array_equal(oracle.count_tiles(r, "2d", k), g["cfg1_counts_r"])
    assert np.array_equal(oracle.count_tiles(s, "2d", k), g["cfg1_counts_s"])


def test_oracle_thread_invariance():
    r, s, k = make_config(1, 0.3)
    base = oracle.sorted_pairs(oracle.join(r, s, "2d", k, threads=1)["pairs"])
    for m in (2, 3, 8):
        got = oracle.sorted_pairs(oracle.join(r, s, "2d", k, threads=m)["pairs"])
        assert np.array_equal(got, base)


def test_generators_reproduce_survey_assignment_counts():
    # exact A_R / A_S of the full-size cfg1 inputs
    r, s, k = make_config(1)
    spec = CONFIGS[1]
    assert int(oracle.count_tiles(r, "2d", k).sum()) == spec.a_r
    assert int(oracle.count_tiles(s, "2d", k).sum()) == spec.a_s
