#!/usr/bin/env python
"""Per-phase device times of run_join with explicit options (experiments).
usage: phase_probe.py [--config 2] [--reps 10] [--bin-bytes N] [--nested-max N]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import CONFIGS, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--bin-bytes", type=int, default=None)
ap.add_argument("--nested-max", type=int, default=-1)
ap.add_argument("--per-rep", action="store_true", help="also print each join's device time")
ap.add_argument("--gc-freeze", action="store_true", help="gc.freeze() after the warm-up")
a = ap.parse_args()
r, s, k = make_config(a.config, 1.0)
R = dev.to_device(r, "cuda")
S = R if s is r else dev.to_device(s, "cuda")
for _ in range(3):
    dev.run_join(R, S, k, k, bin_bytes=a.bin_bytes, nested_max=a.nested_max)
if a.gc_freeze:
    import gc
    gc.collect()
    gc.freeze()
ms0 = torch.cuda.memory_stats()
probe = dev.PhaseProbe()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
t0.record()
for _ in range(a.reps):
    res = dev.run_join(R, S, k, k, probe=probe, bin_bytes=a.bin_bytes, nested_max=a.nested_max)
t1.record()
t1.synchronize()
ph = {n: round(v / a.reps * 1e3, 3) for n, v in probe.durations().items()}
ms1 = torch.cuda.memory_stats()
ph["cudaMalloc/free"] = (ms1.get("num_device_alloc", 0) - ms0.get("num_device_alloc", 0),
                         ms1.get("num_device_free", 0) - ms0.get("num_device_free", 0),
                         ms1.get("num_alloc_retries", 0) - ms0.get("num_alloc_retries", 0))
if a.per_rep:
    reps = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.run_join(R, S, k, k, bin_bytes=a.bin_bytes, nested_max=a.nested_max)
        e1.record()
        e1.synchronize()
        reps.append(round(e0.elapsed_time(e1), 3))
    print("per-rep ms", reps)
print(CONFIGS[a.config].name, f"bin_bytes={a.bin_bytes}", f"{t0.elapsed_time(t1) / a.reps:.3f} ms",
      res.count, ph)
