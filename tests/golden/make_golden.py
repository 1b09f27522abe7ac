"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory under /tmp, builds the
reference's compiled backend there (``setup.py build_ext --inplace``; falls
back to its pure-Python backend if that fails), imports ``sweepjoin`` from the
scratch copy and records the reference's own outputs on seeded inputs:

* ``instances.npz``  — random small instances (mixed extents, degenerate
  points, coordinates snapped to tile boundaries, empty sides, self-joins)
  × layouts; inputs and the reference's sorted pair lists;
* ``configs.npz``    — BASELINE cfg1 at full size and cfg2–5 scaled down:
  result_count, A_R/A_S (PartitionedDataset.total_assigned) and sorted pairs;
* ``tile_of.npz``    — axis_tile_index known answers at and around i/k;
* ``epsilon.npz``    — epsilon_distance_join known answers;
* ``synthetic.npz``  — generate_synthetic outputs, a join of two of them and
  the acceptance criterion-3 count (``python make_golden.py synthetic``);
* ``partition.npz``  — partition() PartitionedDataset arrays (offsets, ids,
  coordinates) for 1D x / 1D y / 2D layouts at m = 1 and m = 3, and
  build_task_queue's sort/join task lists (``python make_golden.py partition``).

Nothing here runs on the GPU box; the .npz files are committed.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from paper_1908_11740_b200.synth import CONFIGS, make_config  # noqa: E402

REFERENCE = Path("/root/reference/pkg")


def import_reference():
    scratch = Path(tempfile.mkdtemp(prefix="sweepjoin_ref_"))
    shutil.copytree(REFERENCE, scratch / "pkg")
    try:
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"],
                       cwd=scratch / "pkg", check=True, capture_output=True)
    except subprocess.CalledProcessError:
        print("warning: compiled backend did not build; using the Python backend")
    sys.path.insert(0, str(scratch / "pkg" / "src"))
    import sweepjoin  # noqa: F401
    print("reference backends:", sweepjoin.available_backends())
    return sweepjoin


def sorted_pairs(p):
    p = np.asarray(p, dtype=np.int64).reshape(-1, 2)
    return p[np.lexsort((p[:, 1], p[:, 0]))] if len(p) else p


def rand_side(rng, n, k_snap, id_base):
    """Uniform centres, exponential extents, some points, some boundary-snapped."""
    scale = float(rng.choice([0.0, 0.002, 0.02, 0.08, 0.3]))
    cx, cy = rng.random(n), rng.random(n)
    ex = rng.exponential(scale, n) if scale > 0 else np.zeros(n)
    ey = rng.exponential(scale, n) if scale > 0 else np.zeros(n)
    pts = rng.random(n) < 0.3
    ex[pts] = 0.0
    ey[pts] = 0.0
    xl, xu = np.clip(cx - ex / 2, 0, 1), np.clip(cx + ex / 2, 0, 1)
    yl, yu = np.clip(cy - ey / 2, 0, 1), np.clip(cy + ey / 2, 0, 1)
    # snap a fraction of coordinates exactly onto tile boundaries i/k (and 0, 1)
    for arr in (xl, xu, yl, yu):
        m = rng.random(n) < 0.25
        arr[m] = np.floor(arr[m] * k_snap) / k_snap
    xl, xu = np.minimum(xl, xu), np.maximum(xl, xu)
    yl, yu = np.minimum(yl, yu), np.maximum(yl, yu)
    return np.arange(id_base, id_base + n, dtype=np.int64), xl, xu, yl, yu


LAYOUTS = [("2d", 1, 0), ("2d", 2, 0), ("2d", 4, 0), ("2d", 7, 0), ("2d", 32, 0),
           ("2d", 100, 0), ("1d", 4, 0), ("1d", 32, 0), ("1d", 16, 1)]


def make_instances(sj, n_inst=48, seed=20261019):
    rng = np.random.default_rng(seed)
    out = {}
    cases = []
    for i in range(n_inst):
        kind, k, axis = LAYOUTS[i % len(LAYOUTS)]
        n_r = int(rng.integers(0 if i % 16 == 5 else 1, 300))
        n_s = int(rng.integers(1, 300))
        snap = int(rng.choice([k, 2 * k, 3])) if k > 1 else 4
        r = rand_side(rng, n_r, snap, 0)
        self_join = i % 12 == 7
        s = r if self_join else rand_side(rng, n_s, snap, 1_000_000)
        R = sj.RectBatch(*r)
        S = R if self_join else sj.RectBatch(*s)
        lay = sj.PartitionLayout(kind, k, sj.Axis(axis))
        rep = sj.join(R, S, sj.JoinConfig(lay, sink_mode="collect-pairs", threads=2))
        truth = sj.nested_loop_join(R, S)
        assert rep.result_count == len(truth)
        assert set(map(tuple, rep.pairs.tolist())) == truth
        tag = f"i{i:03d}"
        for name, arr in zip(("ids", "xl", "xu", "yl", "yu"), r):
            out[f"{tag}_r_{name}"] = arr
        for name, arr in zip(("ids", "xl", "xu", "yl", "yu"), s):
            out[f"{tag}_s_{name}"] = arr
        out[f"{tag}_pairs"] = sorted_pairs(rep.pairs)
        cases.append((tag, kind, k, axis, int(self_join), rep.result_count))
    out["cases"] = np.array([f"{t},{kd},{k},{a},{sj_},{c}" for t, kd, k, a, sj_, c in cases])
    np.savez_compressed(HERE / "instances.npz", **out)
    print("instances:", len(cases))


SCALES = {1: 1.0, 2: 0.01, 3: 0.005, 4: 0.01, 5: 0.02}


def make_configs(sj):
    out = {}
    for cfg, scale in SCALES.items():
        r, s, k = make_config(cfg, scale)
        R = sj.RectBatch(*r)
        S = R if s is r else sj.RectBatch(*s)
        lay = sj.PartitionLayout("2d", k)
        rep = sj.join(R, S, sj.JoinConfig(lay, axis_policy="x", sink_mode="collect-pairs"))
        pr = sj.partition(R, lay)
        ps = sj.partition(S, lay)
        out[f"cfg{cfg}_scale"] = np.float64(scale)
        out[f"cfg{cfg}_count"] = np.int64(rep.result_count)
        out[f"cfg{cfg}_a_r"] = np.int64(pr.total_assigned)
        out[f"cfg{cfg}_a_s"] = np.int64(ps.total_assigned)
        out[f"cfg{cfg}_pairs"] = sorted_pairs(rep.pairs)
        if cfg == 1:
            out["cfg1_counts_r"] = pr.counts.astype(np.int32)
            out["cfg1_counts_s"] = ps.counts.astype(np.int32)
        print(f"cfg{cfg} scale {scale}: P={rep.result_count} A_R={pr.total_assigned} "
              f"A_S={ps.total_assigned}")
    np.savez_compressed(HERE / "configs.npz", **out)


def make_tile_of(sj):
    ps, ks, ts = [], [], []
    for k in (1, 2, 3, 7, 10, 49, 100, 999, 1000, 2000, 3000, 4000, 9973, 20000):
        i = np.arange(0, k + 1)
        if k > 600:  # every boundary of the small grids, a sample of the large ones
            i = np.unique(np.concatenate([i[:100], i[-100:],
                                          np.random.default_rng(k).choice(i, 300)]))
        b = i / k
        for p in np.concatenate([b, np.nextafter(b, -1.0), np.nextafter(b, 2.0),
                                 np.random.default_rng(k).random(64)]):
            if 0.0 <= p <= 1.0:
                ps.append(p)
                ks.append(k)
                ts.append(sj.axis_tile_index(float(p), k))
    np.savez_compressed(HERE / "tile_of.npz", p=np.array(ps), k=np.array(ks),
                        tile=np.array(ts))
    print("tile_of KATs:", len(ps))


def make_epsilon(sj):
    rng = np.random.default_rng(77)
    out = {}
    for i, (n, eps, k) in enumerate([(400, 0.02, 16), (300, 0.05, 8), (500, 1e-3, 100)]):
        x, y = rng.random(n), rng.random(n)
        # a few exact-distance ties on the eps circle
        x[:10] = np.clip(x[10:20] + eps, 0, 1)
        y[:10] = y[10:20]
        P = sj.RectBatch(np.arange(n, dtype=np.int64), x, x, y, y)
        x2, y2 = rng.random(n), rng.random(n)
        Q = sj.RectBatch(np.arange(n, dtype=np.int64) + 5000, x2, x2, y2, y2)
        rep = sj.epsilon_distance_join(P, Q, eps, sj.JoinConfig(
            sj.PartitionLayout("2d", k), sink_mode="collect-pairs"))
        out[f"e{i}_p"] = np.stack([x, y])
        out[f"e{i}_q"] = np.stack([x2, y2])
        out[f"e{i}_eps"] = np.float64(eps)
        out[f"e{i}_k"] = np.int64(k)
        out[f"e{i}_pairs"] = sorted_pairs(rep.pairs)
    np.savez_compressed(HERE / "epsilon.npz", **out)


SYNTH_SPECS = [  # (name, SyntheticSpec kwargs); ids are row indices
    ("u", dict(n=4000, x_extent_mean=2e-3, y_extent_mean=2e-3, seed=11)),
    ("g", dict(n=3000, x_extent_mean=5e-3, y_extent_mean=1e-3,
               distribution="gaussian-clustered", seed=12, clusters=8, cluster_sigma=0.03)),
    ("p", dict(n=2000, seed=13)),  # points
]


def make_synthetic(sj):
    """The reference's generate_synthetic outputs (pins synth.synthetic), the
    join of two of them (pairs), and the acceptance criterion-3 instance's
    count (SyntheticSpec(1_000_000, 1e-3, 1e-3, seed 301 / 302), 1D K=100)."""
    from sweepjoin.io import SyntheticSpec, generate_synthetic
    out = {}
    for name, kw in SYNTH_SPECS:
        b = generate_synthetic(SyntheticSpec(**kw))
        for c in ("ids", "xl", "xu", "yl", "yu"):
            out[f"{name}_{c}"] = getattr(b, c)
    r = generate_synthetic(SyntheticSpec(**SYNTH_SPECS[0][1]))
    s = generate_synthetic(SyntheticSpec(**SYNTH_SPECS[1][1]))
    rep = sj.join(r, s, sj.JoinConfig(sj.PartitionLayout("2d", 32), sink_mode="collect-pairs"))
    out["ug_k32_pairs"] = sorted_pairs(rep.pairs)
    r = generate_synthetic(SyntheticSpec(1_000_000, 1e-3, 1e-3, seed=301))
    s = generate_synthetic(SyntheticSpec(1_000_000, 1e-3, 1e-3, seed=302))
    rep = sj.join(r, s, sj.JoinConfig(sj.PartitionLayout("1d", 100), threads=os.cpu_count() or 1))
    out["crit3_count"] = np.int64(rep.result_count)
    print("criterion-3 count:", rep.result_count)
    np.savez_compressed(HERE / "synthetic.npz", **out)


PART_LAYOUTS = [("1d", 7, 0), ("1d", 6, 1), ("2d", 5, 0), ("2d", 23, 0)]


def make_partition(sj):
    """partition() (partition.py:243-263) and build_task_queue
    (engine.py:84-100) known answers on seeded mixed-extent inputs."""
    from sweepjoin.partition import partition
    rng = np.random.default_rng(2024)
    out = {}
    for i in range(2):
        n = 600 + 200 * i
        xl, yl = rng.random(n), rng.random(n)
        w = np.where(rng.random(n) < 0.2, rng.random(n) * 0.5, rng.random(n) * 0.02)
        h = np.where(rng.random(n) < 0.2, rng.random(n) * 0.5, rng.random(n) * 0.02)
        xl[:20] = np.round(xl[:20] * 5) / 5   # on tile boundaries of K=5
        batch = sj.RectBatch(np.arange(n, dtype=np.int64) * 3 + 1, xl, np.minimum(xl + w, 1.0),
                             yl, np.minimum(yl + h, 1.0))
        for c in ("ids", "xl", "xu", "yl", "yu"):
            out[f"p{i}_{c}"] = getattr(batch, c)
        for j, (kind, k, axis) in enumerate(PART_LAYOUTS):
            layout = sj.PartitionLayout(kind, k, sj.Axis(axis))
            for m in (1, 3):
                pd = partition(batch, layout, m=m)
                tag = f"p{i}_l{j}_m{m}"
                out[f"{tag}_offsets"] = pd.offsets
                for c in ("ids", "xl", "xu", "yl", "yu"):
                    out[f"{tag}_{c}"] = getattr(pd, c)
        # task queue of input 0 vs input 1 on the 2D K=5 layout
    layout = sj.PartitionLayout("2d", 5)
    pr = partition(sj.RectBatch(*(out[f"p0_{c}"] for c in ("ids", "xl", "xu", "yl", "yu"))),
                   layout)
    ps = partition(sj.RectBatch(*(out[f"p1_{c}"] for c in ("ids", "xl", "xu", "yl", "yu"))),
                   layout)
    sort_tasks, join_tasks = sj.build_task_queue(pr, ps)
    out["tq_sort"] = np.array([tuple(t) for t in sort_tasks], dtype=np.int64)
    out["tq_join"] = np.array([tuple(t) for t in join_tasks], dtype=np.int64)
    out["layouts"] = np.array([f"{a},{b},{c}" for a, b, c in PART_LAYOUTS])
    np.savez_compressed(HERE / "partition.npz", **out)


if __name__ == "__main__":
    sj = import_reference()
    if sys.argv[1:] == ["synthetic"]:
        make_synthetic(sj)
        sys.exit(0)
    if sys.argv[1:] == ["partition"]:
        make_partition(sj)
        sys.exit(0)
    make_tile_of(sj)
    make_instances(sj)
    make_epsilon(sj)
    make_configs(sj)
    make_synthetic(sj)
    make_partition(sj)
