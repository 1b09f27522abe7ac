"""Larger parity anchors for the round-2 API surface, computed by the REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_extra_truth.py

* ``eps_*``: ``sweepjoin.epsilon_distance_join`` (engine.py:326-353) on the
  points cfg4's squares are built from (``synth.cfg4_points``: R uniform,
  S a 128-cluster mixture) at reduced size, and one self-join — the count,
  the candidate (square-join) count and the sha256 of the sorted pair list;
* ``part_*``: ``sweepjoin.partition`` (partition.py:243-263) of cfg1's R
  (2D K=100) and cfg5's R (1D stripes along y, K=1000) — total_assigned and
  the sha256 of every PartitionedDataset array (offsets, ids, xl, xu, yl, yu).

Inputs are regenerated from seeds by the tests; only the answers are
committed (``extra_truth.json``).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

from make_golden import import_reference, sorted_pairs  # noqa: E402

from paper_1908_11740_b200.synth import cfg4_points, make_config  # noqa: E402

OUT = HERE / "extra_truth.json"
EPS_CASES = {  # name: (n per side, eps, K, self-join)
    "eps_cfg4_400k": (400_000, 1e-3, 400, False),
    "eps_cfg4_1m_fine": (1_000_000, 2.5e-4, 1000, False),
    "eps_self_300k": (300_000, 1e-3, 300, True),
}
PART_CASES = {  # name: (cfg, kind, k, axis)
    "part_cfg1_2d": (1, "2d", 100, 0),
    "part_cfg5_1dy": (5, "1d", 1000, 1),
}


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def eps_inputs(name):
    n, eps, k, self_join = EPS_CASES[name]
    p = cfg4_points(n, 0, False)
    q = p if self_join else cfg4_points(n, 1, True)
    return p, q, eps, k


def part_input(name):
    cfg, kind, k, axis = PART_CASES[name]
    r, _, _ = make_config(cfg, 0.2 if cfg == 5 else 1.0)
    return r, kind, k, axis


def main():
    sj = import_reference()
    out = {}
    for name in EPS_CASES:
        t0 = time.perf_counter()
        (pi, px, py), q, eps, k = eps_inputs(name)
        P = sj.RectBatch(pi, px, px, py, py)
        Q = P if q[0] is pi else sj.RectBatch(q[0], q[1], q[1], q[2], q[2])
        cfg = sj.JoinConfig(sj.PartitionLayout("2d", k), axis_policy="x",
                            sink_mode="collect-pairs", threads=8)
        rep = sj.epsilon_distance_join(P, Q, eps, cfg)
        pairs = np.ascontiguousarray(sorted_pairs(rep.pairs), dtype="<i8")
        out[name] = {"count": int(rep.result_count), "pairs_sha256": sha(pairs),
                     "n": EPS_CASES[name][0], "eps": eps, "k": k,
                     "self_join": EPS_CASES[name][3],
                     "reference_s": round(time.perf_counter() - t0, 3)}
        print(name, out[name], flush=True)
    for name in PART_CASES:
        r, kind, k, axis = part_input(name)
        pd = sj.partition(sj.RectBatch(*r), sj.PartitionLayout(kind, k, sj.Axis(axis)))
        out[name] = {"total_assigned": int(pd.total_assigned),
                     "sha256": sha(pd.offsets.astype("<i8"), pd.ids.astype("<i8"),
                                   pd.xl.astype("<f8"), pd.xu.astype("<f8"),
                                   pd.yl.astype("<f8"), pd.yu.astype("<f8")),
                     "kind": kind, "k": k, "axis": axis}
        print(name, out[name], flush=True)
    OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
