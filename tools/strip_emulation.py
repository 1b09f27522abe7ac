"""Projected N-GPU step of bench.py from one GPU: each rank's strip join
(the same strip plan, inputs and run_join call as bench.py at --gpus N) timed
ALONE on cuda:0, one strip after another — the strips share nothing, so the
N-GPU step is the slowest strip plus the count all_gather (not included).
Not a multi-GPU measurement: a projection of what one would see.

usage: python tools/strip_emulation.py [--config 2] [--ns 2 4 8] [--steps 10]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import device as dev, parallel  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--ns", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
r, s, k = make_config(a.config)
self_join = s is r
n_tot = len(r[0]) + len(s[0])
for n in a.ns:
    plan = parallel.plan_strips(r, s, k, n)
    per = []
    for g in range(n):
        lo, hi = plan[g], plan[g + 1]
        rr = parallel.strip_inputs(r, k, lo, hi)
        ss = rr if self_join else parallel.strip_inputs(s, k, lo, hi)
        rd = dev.to_device(rr, "cuda")
        sd = rd if self_join else dev.to_device(ss, "cuda")
        for _ in range(3):
            res = dev.run_join(rd, sd, k, k, collect=True, row_lo=lo, row_hi=hi, graph=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            res = dev.run_join(rd, sd, k, k, collect=True, row_lo=lo, row_hi=hi, graph=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        probe = dev.PhaseProbe()
        for _ in range(a.steps):
            dev.run_join(rd, sd, k, k, collect=True, row_lo=lo, row_hi=hi, probe=probe)
        torch.cuda.synchronize()
        ph = {k_: round(v / a.steps * 1e3, 4) for k_, v in probe.durations().items()
              if k_ != "start"}
        per.append({"rows": [lo, hi], "n_r": len(rr[0]), "n_s": len(ss[0]), "ms": round(ms, 4),
                    "pairs": res.count, "a_r": res.header["a_r"], "a_s": res.header["a_s"],
                    "max_tile": res.header.get("max_tile"), "phases_ms": ph})
        del rd, sd, res
        dev.release_buffers()
    t = max(p["ms"] for p in per)
    print(json.dumps({"config": a.config, "n": n, "projected_ms": t,
                      "projected_rects_per_s": n_tot / (t / 1e3),
                      "mean_ms": sum(p["ms"] for p in per) / n, "strips": per}), flush=True)
