"""cProfile of the host side of near-empty joins (the fixed per-join cost)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402

n, k = 1000, int(sys.argv[1]) if len(sys.argv) > 1 else 100


def rects(seed):
    g = np.random.default_rng(seed)
    xl, yl = g.random(n), g.random(n)
    return (np.arange(n, dtype=np.int64), xl, np.minimum(xl + 1e-4, 1.0), yl,
            np.minimum(yl + 1e-4, 1.0))


R, S = dev.to_device(rects(0)), dev.to_device(rects(1))
for _ in range(10):
    dev.run_join(R, S, k, k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    dev.run_join(R, S, k, k)
print("wall us/join", (time.perf_counter() - t0) / 200 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    dev.run_join(R, S, k, k)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
