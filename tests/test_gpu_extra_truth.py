"""GPU parity at larger sizes for the round-2 API surface, against answers the
REFERENCE computed (tests/golden/extra_truth.json, make_extra_truth.py):
the fused ε-distance join on cfg4's points (two sizes, one self-join) and
partition() on cfg1 / cfg5 inputs.  Inputs are regenerated from the seeds."""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
import paper_1908_11740_b200 as pb

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))
TRUTH = json.loads((HERE / "golden" / "extra_truth.json").read_text())


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    torch.cuda.set_device(0)


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", [n for n in TRUTH if n.startswith("eps_")])
def test_fused_epsilon_join_vs_reference_truth(name):
    from make_extra_truth import eps_inputs

    (pi, px, py), q, eps, k = eps_inputs(name)
    P = pb.RectBatch(pi, px, px, py, py)
    Q = P if q[0] is pi else pb.RectBatch(q[0], q[1], q[1], q[2], q[2])
    rep = pb.epsilon_distance_join(P, Q, eps, pb.JoinConfig(pb.PartitionLayout("2d", k),
                                                             sink_mode="collect-pairs"))
    t = TRUTH[name]
    assert rep.result_count == t["count"]
    got = np.ascontiguousarray(oracle.sorted_pairs(rep.pairs), dtype="<i8")
    assert _sha(got) == t["pairs_sha256"]


@pytest.mark.parametrize("name", [n for n in TRUTH if n.startswith("part_")])
def test_partition_vs_reference_truth(name):
    from make_extra_truth import part_input

    r, kind, k, axis = part_input(name)
    pd = pb.partition(pb.RectBatch(*r), pb.PartitionLayout(kind, k, pb.Axis(axis)))
    t = TRUTH[name]
    assert pd.total_assigned == t["total_assigned"]
    assert _sha(pd.offsets.astype("<i8"), pd.ids.astype("<i8"), pd.xl.astype("<f8"),
                pd.xu.astype("<f8"), pd.yl.astype("<f8"), pd.yu.astype("<f8")) == t["sha256"]
