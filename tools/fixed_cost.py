"""Fixed per-join cost: device time of near-empty joins (n rectangles per
input) on several grids / strips, through run_join (the repeated-shape,
speculative path after warm-up), with the phase split.
usage: python tools/fixed_cost.py [n]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(0)


def rects(seed):
    g = np.random.default_rng(seed)
    xl, yl = g.random(n), g.random(n)
    return (np.arange(n, dtype=np.int64), xl, np.minimum(xl + 1e-4, 1.0), yl,
            np.minimum(yl + 1e-4, 1.0))


R, S = dev.to_device(rects(0)), dev.to_device(rects(1))
torch.cuda.synchronize()
graph = len(sys.argv) > 2 and sys.argv[2] == "graph"
for k, lo, hi in [(100, 0, 100), (2000, 0, 2000), (2000, 0, 250), (2000, 1000, 1250),
                  (4000, 0, 500)]:
    for _ in range(5):
        dev.run_join(R, S, k, k, row_lo=lo, row_hi=hi, graph=graph)
    torch.cuda.synchronize()
    steps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        res = dev.run_join(R, S, k, k, row_lo=lo, row_hi=hi, graph=graph)
    e1.record()
    torch.cuda.synchronize()
    probe = dev.PhaseProbe()
    for _ in range(steps):
        dev.run_join(R, S, k, k, row_lo=lo, row_hi=hi, probe=probe)
    torch.cuda.synchronize()
    ph = {a: round(b / steps * 1e6, 1) for a, b in probe.durations().items()}
    print(json.dumps({"graph": graph, "k": k, "rows": [lo, hi], "n": n, "us_per_join":
                      round(e0.elapsed_time(e1) / steps * 1e3, 1), "pairs": res.count,
                      "phases_us": ph}), flush=True)
