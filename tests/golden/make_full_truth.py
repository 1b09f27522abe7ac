"""Full-size truth for BASELINE configs 1-5, computed by the REFERENCE itself.

Run in the build container (where /root/reference exists; minutes per config):

    python tests/golden/make_full_truth.py [cfg ...]

For every config it builds the reference's compiled backend in a scratch copy
(``make_golden.import_reference``), generates the full-size inputs with
``synth.make_config`` (the SURVEY.md §8(d) numpy recipe), runs

    sweepjoin.join(R, S, JoinConfig(PartitionLayout("2d", K), axis_policy="x",
                                    sink_mode="collect-pairs", threads=1))

(engine.py:312-323) and ``sweepjoin.partition`` for A_R / A_S
(PartitionedDataset.total_assigned, partition.py:101-103), and records
``result_count``, A_R, A_S and the sha256 of the lexicographically sorted
(r_id, s_id) int64 pair list (C order, little-endian: ``pairs_sha256``).
The records go to ``tests/golden/full_truth.json`` (committed); the GPU
tests and ``bench.py``'s parity gate compare against these hashes, so the
full-size parity claims no longer rest on survey constants.
"""

from __future__ import annotations

import hashlib
import json
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

from make_golden import import_reference, sorted_pairs  # noqa: E402

from paper_1908_11740_b200.synth import make_config  # noqa: E402

OUT = HERE / "full_truth.json"


def pairs_sha256(pairs: np.ndarray) -> str:
    p = np.ascontiguousarray(sorted_pairs(pairs), dtype="<i8")
    return hashlib.sha256(p.tobytes()).hexdigest()


def main(cfgs):
    sj = import_reference()
    truth = json.loads(OUT.read_text()) if OUT.exists() else {}
    for cfg in cfgs:
        t0 = time.perf_counter()
        r, s, k = make_config(cfg)
        R = sj.RectBatch(*r)
        S = R if s is r else sj.RectBatch(*s)
        lay = sj.PartitionLayout("2d", k)
        rep = sj.join(R, S, sj.JoinConfig(lay, axis_policy="x", sink_mode="collect-pairs",
                                          threads=1))
        digest = pairs_sha256(rep.pairs)
        n_pairs = int(len(rep.pairs))
        join_s = rep.total_time
        del rep
        a_r = int(sj.partition(R, lay).total_assigned)
        a_s = a_r if S is R else int(sj.partition(S, lay).total_assigned)
        truth[f"cfg{cfg}"] = {
            "n_r": len(r[0]), "n_s": len(s[0]), "k": k, "self_join": s is r,
            "count": n_pairs, "a_r": a_r, "a_s": a_s, "pairs_sha256": digest,
            "reference_total_time_s": round(join_s, 3),
            "reference_call": "sweepjoin.join(R, S, JoinConfig(PartitionLayout('2d', K), "
                              "axis_policy='x', sink_mode='collect-pairs', threads=1))",
            "host": f"{platform.machine()} {platform.processor() or ''}".strip(),
        }
        print(f"cfg{cfg}: P={n_pairs} A_R={a_r} A_S={a_s} sha256={digest[:16]}... "
              f"(reference join {join_s:.1f} s, wall {time.perf_counter() - t0:.1f} s)",
              flush=True)
        OUT.write_text(json.dumps(truth, indent=2, sort_keys=True) + "\n")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 5, 3, 4])
