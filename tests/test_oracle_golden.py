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


def test_synthetic_generator_matches_reference(golden):
    """synth.synthetic restates the reference's generate_synthetic (io.py:189-227)
    byte for byte (fixtures from the reference itself)."""
    from paper_1908_11740_b200.synth import synthetic
    g = golden["synthetic"]
    for name, kw in _synth_specs():
        got = synthetic(**kw)
        for c, a in zip(("ids", "xl", "xu", "yl", "yu"), got):
            assert np.array_equal(a, g[f"{name}_{c}"]), (name, c)


def _synth_specs():
    # the specs of tests/golden/make_golden.py SYNTH_SPECS
    return [
        ("u", dict(n=4000, x_extent_mean=2e-3, y_extent_mean=2e-3, seed=11)),
        ("g", dict(n=3000, x_extent_mean=5e-3, y_extent_mean=1e-3,
                   distribution="gaussian-clustered", seed=12, clusters=8, cluster_sigma=0.03)),
        ("p", dict(n=2000, seed=13)),
    ]


def test_oracle_synthetic_join_and_criterion3(golden):
    """The oracle on the reference's synthetic workloads: the u x g join's pairs,
    and the acceptance criterion-3 instance (1M x 1M, 1D K=100) count."""
    from paper_1908_11740_b200.synth import synthetic
    g = golden["synthetic"]
    specs = dict(_synth_specs())
    res = oracle.join(synthetic(**specs["u"]), synthetic(**specs["g"]), "2d", 32)
    assert np.array_equal(oracle.sorted_pairs(res["pairs"]), g["ug_k32_pairs"])
    r = synthetic(1_000_000, 1e-3, 1e-3, seed=301)
    s = synthetic(1_000_000, 1e-3, 1e-3, seed=302)
    res = oracle.join(r, s, "1d", 100, threads=8, collect=False)
    assert res["count"] == int(g["crit3_count"]) == 3_989_612


def test_full_truth_is_consistent_with_fixtures():
    """tests/golden/full_truth.json (the reference's full-size outputs, made by
    make_full_truth.py) agrees with the committed cfg1 pair fixture (hash of
    the same sorted list) and with the survey's A_R / A_S / P constants."""
    import hashlib
    import json
    from pathlib import Path

    import numpy as np

    from paper_1908_11740_b200.synth import CONFIGS

    truth = json.loads((Path(__file__).resolve().parent / "golden" / "full_truth.json")
                       .read_text())
    g = np.load(Path(__file__).resolve().parent / "golden" / "configs.npz")
    p = np.ascontiguousarray(g["cfg1_pairs"], dtype="<i8")
    assert hashlib.sha256(p.tobytes()).hexdigest() == truth["cfg1"]["pairs_sha256"]
    for name, t in truth.items():
        spec = CONFIGS[int(name[3:])]
        assert (t["count"], t["a_r"], t["a_s"]) == (spec.pairs, spec.a_r, spec.a_s), name
        assert (t["n_r"], t["n_s"], t["k"]) == (spec.n_r, spec.n_s, spec.k), name


def test_oracle_epsilon_join_matches_reference(golden):
    # the CPU restatement of epsilon_distance_join (engine.py:326-353) vs the
    # reference's own outputs
    g = golden["epsilon"]
    for i in range(3):
        x, y = g[f"e{i}_p"]
        x2, y2 = g[f"e{i}_q"]
        n = len(x)
        P = (np.arange(n, dtype=np.int64), x, x, y, y)
        Q = (np.arange(n, dtype=np.int64) + 5000, x2, x2, y2, y2)
        res = oracle.epsilon_join(P, Q, float(g[f"e{i}_eps"]), int(g[f"e{i}_k"]))
        assert np.array_equal(oracle.sorted_pairs(res["pairs"]), g[f"e{i}_pairs"])
        assert res["candidates"] >= res["count"]
