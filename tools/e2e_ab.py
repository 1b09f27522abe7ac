"""A/B of the end-to-end join() path in one process (same pinned inputs,
modes interleaved, median of each): staged return on/off and id group counts.
usage: python tools/e2e_ab.py [--config 2] [--reps 9]"""
import argparse
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import JoinConfig, PartitionLayout, RectBatch, engine  # noqa: E402
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=9)
a = ap.parse_args()
r, s, k = make_config(a.config)


def pinned(b):
    out = []
    for x in b:
        t = torch.empty(x.shape, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True)
        t.numpy()[:] = x
        out.append(t.numpy())
    return RectBatch(*out)


R = pinned(r)
S = R if s is r else pinned(s)
cfg = JoinConfig(PartitionLayout("2d", k), sink_mode="collect-pairs")
modes = {"unstaged": (False, 8), "staged4": (True, 4), "staged8": (True, 8),
         "staged16": (True, 16)}
times = {m: [] for m in modes}
for rep in range(a.reps + 1):
    for m, (st, g) in modes.items():
        dev.STAGED, dev.ID_GROUPS = st, g
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = engine.join(R, S, cfg)
        dt = time.perf_counter() - t0
        if rep:
            times[m].append(dt * 1e3)
for m, v in times.items():
    print(f"{m:10s} median {statistics.median(v):7.3f} ms  min {min(v):7.3f}  max {max(v):7.3f}")
