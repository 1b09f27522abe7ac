"""One pass over every kernel of the library, for `ncu --set full` captures
(tools/gpu/ncu_all.sh): the cfg2 join (eager launches), a cfg4 join with the
binned scatter, a host-input join (id map + pair groups), the fused ε-join,
the huge-tile sort + sweep, the pair sort, strip routing, partition() and the
SJB1 device loader.  Each workload runs 3 times so --kernel-id ...:3 sees a
warm launch of each kernel."""
import sys
import tempfile
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1908_11740_b200 as pb  # noqa: E402
from paper_1908_11740_b200 import device as dev, io, parallel  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
torch.cuda.set_device(0)


def rep(fn, n=3):
    for _ in range(n):
        fn()
    torch.cuda.synchronize()


if which in ("all", "cfg2"):
    r, s, k = make_config(2)
    R, S = dev.to_device(r), dev.to_device(s)
    rep(lambda: dev.run_join(R, S, k, k))
    res = dev.run_join(R, S, k, k)
    rep(lambda: parallel.canonical_pairs(res.pairs))
    cuts = parallel.plan_strips(r, s, k, 8)
    rep(lambda: parallel._route_device(R.columns(), k, cuts))
    del R, S, res
    dev.release_buffers()
if which in ("all", "cfg4"):
    r, s, k = make_config(4)
    R, S = dev.to_device(r), dev.to_device(s)
    rep(lambda: dev.run_join(R, S, k, k))  # (cfg4's lists take the binned scatter)
    del R, S
    dev.release_buffers()
if which in ("all", "misc"):
    r, s, k = make_config(2, 0.1)
    cfg = pb.JoinConfig(pb.PartitionLayout("2d", k), sink_mode="collect-pairs")
    rep(lambda: pb.join(pb.RectBatch(*r), pb.RectBatch(*s), cfg))  # staged return
    P = pb.RectBatch(r[0], r[1], r[1], r[3], r[3])
    Q = pb.RectBatch(s[0], s[1], s[1], s[3], s[3])
    rep(lambda: pb.epsilon_distance_join(P, Q, 2e-4, cfg))
    n = 60000  # one huge tile: sort + forward-scan sweep
    g = np.random.default_rng(0)
    xl = g.random(n) * 0.5
    yl = g.random(n) * 0.5
    big = (np.arange(n, dtype=np.int64), xl, xl + 1e-3, yl, yl + 1e-3)
    B = dev.to_device(big)
    rep(lambda: dev.run_join(B, B, 2, 2, sweep_min=0))
    rep(lambda: pb.partition(pb.RectBatch(*r), pb.PartitionLayout("2d", k)))
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "r.sjb1"
        io.save_mbr_binary(pb.RectBatch(*r), f)
        rep(lambda: io.load_dataset_device(f))
if which == "misc2":  # the instances misc does not reach: ε-join, routing pack, pair groups
    r, s, k = make_config(2, 0.3)
    cfg = pb.JoinConfig(pb.PartitionLayout("2d", k), sink_mode="collect-pairs")
    rep(lambda: pb.join(pb.RectBatch(*r), pb.RectBatch(*s), cfg))  # staged return: groups
    P = pb.RectBatch(r[0], r[1], r[1], r[3], r[3])
    Q = pb.RectBatch(s[0], s[1], s[1], s[3], s[3])
    rep(lambda: pb.epsilon_distance_join(P, Q, 2e-4, cfg))
    R = dev.to_device(r)
    cuts = parallel.plan_strips(r, s, k, 8)
    rep(lambda: parallel._route_device(R.columns(), k, cuts))
print("workload done")
