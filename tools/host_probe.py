#!/usr/bin/env python
"""Host-side cost of one run_join (experiments): wall time per join vs the
device time between its first and last kernel, plus a line profile of the
Python driver.  usage: host_probe.py [--config 2] [--reps 30]"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
r, s, k = make_config(a.config, 1.0)
R = dev.to_device(r, "cuda")
S = R if s is r else dev.to_device(s, "cuda")
for _ in range(3):
    dev.run_join(R, S, k, k)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.reps):
    dev.run_join(R, S, k, k)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / a.reps
probe = dev.PhaseProbe()
for _ in range(a.reps):
    dev.run_join(R, S, k, k, probe=probe)
ph = {n: round(v / a.reps * 1e3, 3) for n, v in probe.durations().items()}
print(f"wall {wall * 1e3:.3f} ms per join; phases {ph}")
pr = cProfile.Profile()
pr.enable()
for _ in range(a.reps):
    dev.run_join(R, S, k, k)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
