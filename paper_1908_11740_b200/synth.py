"""Seeded synthetic MBR generators for the five BASELINE configurations.

The paper measures on TIGER/OSM extracts that are not available here; these
seeded generators stand in for them with the shapes, sizes and value
distributions BASELINE.json states.  The exact numpy call sequence is the one
fixed in SURVEY.md §8(d) (``numpy.random.default_rng`` / PCG64, the generator
the reference itself uses in ``pkg/src/sweepjoin/io.py:210``), so the arrays
are byte-identical to the ones the survey measured A_R, A_S and P on.

Every generator returns ``(ids, xl, xu, yl, yu)`` as C-contiguous int64 /
float64 numpy arrays — the reference ``RectBatch`` column order
(``pkg/src/sweepjoin/geometry.py:109-130``).  ``n`` can be scaled down for
parity tests; the recipe is otherwise unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["CONFIGS", "ConfigSpec", "make_config", "make_side", "synthetic"]


def _clip(a):
    return np.clip(a, 0.0, 1.0)


def _box(cx, cy, w, h):
    return _clip(cx - w / 2), _clip(cx + w / 2), _clip(cy - h / 2), _clip(cy + h / 2)


def _mix(rng, m, n, s0, s1):
    mu = rng.random((m, 2))
    sig = rng.uniform(s0, s1, m)
    pick = rng.integers(0, m, n)
    cx = _clip(mu[pick, 0] + rng.normal(0, 1, n) * sig[pick])
    cy = _clip(mu[pick, 1] + rng.normal(0, 1, n) * sig[pick])
    return cx, cy


def _pack(xl, xu, yl, yu):
    n = len(xl)
    return (np.arange(n, dtype=np.int64),
            np.ascontiguousarray(xl, dtype=np.float64),
            np.ascontiguousarray(xu, dtype=np.float64),
            np.ascontiguousarray(yl, dtype=np.float64),
            np.ascontiguousarray(yu, dtype=np.float64))


def gen_cfg1(n: int, seed: int):
    rng = np.random.default_rng(seed)
    xl = rng.random(n)
    yl = rng.random(n)
    w = rng.uniform(0, 1e-3, n)
    h = rng.uniform(0, 1e-3, n)
    return _pack(xl, np.minimum(xl + w, 1.0), yl, np.minimum(yl + h, 1.0))


def gen_cfg2(n: int, seed: int):
    rng = np.random.default_rng(seed)
    cx, cy = _mix(rng, 64, n, .005, .05)
    w = np.minimum(rng.lognormal(np.log(2e-5), 1.0, n), 1e-2)
    h = np.minimum(rng.lognormal(np.log(2e-5), 1.0, n), 1e-2)
    return _pack(*_box(cx, cy, w, h))


def gen_cfg3(n: int, seed: int):
    rng = np.random.default_rng(seed)
    nn = int(round(0.1 * n))
    cx, cy = _mix(rng, 256, n - nn, .002, .03)
    cx = np.concatenate([cx, rng.random(nn)])
    cy = np.concatenate([cy, rng.random(nn)])
    a = rng.lognormal(np.log(5e-5), 1.0, n)
    b = a * rng.uniform(0.01, 1.0, n)
    f = rng.random(n) < 0.5
    w = np.where(f, a, b)
    h = np.where(f, b, a)
    return _pack(*_box(cx, cy, w, h))


def _squares(px, py, eps=1e-4):
    # engine.py:342-350 arithmetic: half = eps / 2.0, clip(x -/+ half) to [0, 1]
    half = eps / 2.0
    return _pack(_clip(px - half), _clip(px + half), _clip(py - half), _clip(py + half))


def gen_cfg4_r(n: int, seed: int):
    rng = np.random.default_rng(seed)
    px = rng.random(n)
    py = rng.random(n)
    return _squares(px, py)


def gen_cfg4_s(n: int, seed: int):
    rng = np.random.default_rng(seed)
    px, py = _mix(rng, 128, n, .005, .05)
    return _squares(px, py)


def gen_cfg5(n: int, seed: int):
    rng = np.random.default_rng(seed)
    xl = rng.random(n)
    yl = rng.random(n)
    w = np.minimum((rng.pareto(1.5, n) + 1) * 1e-5, 0.05)
    h = np.minimum((rng.pareto(1.5, n) + 1) * 1e-5, 0.05)
    return _pack(xl, np.minimum(xl + w, 1.0), yl, np.minimum(yl + h, 1.0))


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n_r: int
    n_s: int
    k: int
    self_join: bool
    gen_r: object
    gen_s: object
    # exact full-scale values (SURVEY.md §8 header table), re-derived by the
    # reference itself in tests/golden/full_truth.json (make_full_truth.py)
    a_r: int
    a_s: int
    pairs: int


CONFIGS = {
    1: ConfigSpec("cfg1", 100_000, 100_000, 100, False, gen_cfg1, gen_cfg1,
                  110_325, 110_149, 10_101),
    2: ConfigSpec("cfg2", 10_000_000, 10_000_000, 2000, False, gen_cfg2, gen_cfg2,
                  11_312_048, 11_338_579, 2_157_134),
    3: ConfigSpec("cfg3", 20_000_000, 70_000_000, 3000, False, gen_cfg3, gen_cfg3,
                  28_981_295, 101_594_466, 48_512_273),
    4: ConfigSpec("cfg4", 50_000_000, 50_000_000, 4000, False, gen_cfg4_r, gen_cfg4_s,
                  97_984_342, 96_869_277, 97_958_702),
    5: ConfigSpec("cfg5", 5_000_000, 5_000_000, 1000, True, gen_cfg5, gen_cfg5,
                  5_300_431, 5_300_431, 5_089_522),
}


def synthetic(n: int, x_extent_mean: float = 0.0, y_extent_mean: float = 0.0,
              distribution: str = "uniform", seed: int = 0, clusters: int = 16,
              cluster_sigma: float = 0.05):
    """The reference's own synthetic workload (``SyntheticSpec`` /
    ``generate_synthetic``, io.py:189-227), restated: uniform or
    Gaussian-clustered centres, exponentially distributed extents around the
    per-axis means (0 → points), boxes clipped to the unit square, ids =
    row indices.  Used for the reference's acceptance anchors."""
    if n < 0:
        raise ValueError("n must be >= 0")
    if n == 0:
        z = np.empty(0)
        return np.empty(0, dtype=np.int64), z, z.copy(), z.copy(), z.copy()
    rng = np.random.default_rng(seed)
    if distribution == "uniform":
        cx = rng.random(n)
        cy = rng.random(n)
    elif distribution == "gaussian-clustered":
        centres = rng.random((max(1, clusters), 2))
        pick = rng.integers(0, len(centres), n)
        cx = _clip(centres[pick, 0] + rng.normal(0.0, cluster_sigma, n))
        cy = _clip(centres[pick, 1] + rng.normal(0.0, cluster_sigma, n))
    else:
        raise ValueError(f"unknown distribution {distribution!r}")
    ex = rng.exponential(x_extent_mean, n) if x_extent_mean > 0 else np.zeros(n)
    ey = rng.exponential(y_extent_mean, n) if y_extent_mean > 0 else np.zeros(n)
    return (np.arange(n, dtype=np.int64), _clip(cx - ex / 2), _clip(cx + ex / 2),
            _clip(cy - ey / 2), _clip(cy + ey / 2))


def make_side(cfg: int, side: str, n: int | None = None):
    """One input of config ``cfg`` ('r' seed 0, 's' seed 1), optionally resized."""
    spec = CONFIGS[cfg]
    if side == "r":
        return spec.gen_r(spec.n_r if n is None else n, 0)
    if spec.self_join:
        return make_side(cfg, "r", n)
    return spec.gen_s(spec.n_s if n is None else n, 1)


def make_config(cfg: int, scale: float = 1.0):
    """(R, S, K) for config ``cfg`` with both sides scaled by ``scale``."""
    spec = CONFIGS[cfg]
    nr = max(1, int(round(spec.n_r * scale)))
    ns = max(1, int(round(spec.n_s * scale)))
    r = make_side(cfg, "r", nr)
    s = r if spec.self_join else make_side(cfg, "s", ns)
    return r, s, spec.k


def cfg4_points(n: int, seed: int, clustered: bool):
    """The points cfg4's squares are built from: R uniform
    (seed 0), S a 128-cluster mixture (seed 1) — as (ids, px, py) for the
    ε-distance join (which takes the points, engine.py:326-353)."""
    rng = np.random.default_rng(seed)
    if clustered:
        px, py = _mix(rng, 128, n, 0.005, 0.05)
    else:
        px = rng.random(n)
        py = rng.random(n)
    return (np.arange(n, dtype=np.int64), np.ascontiguousarray(px, dtype=np.float64),
            np.ascontiguousarray(py, dtype=np.float64))
