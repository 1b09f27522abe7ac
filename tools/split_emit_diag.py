"""Diagnostic: the compact-entry join with ids NOT gathered at the emit (pairs
hold rows) vs gathered — where the join-side cost of the compact format goes."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
r, s, k = make_config(cfg)
R = dev.to_device(r)
S = R if s is r else dev.to_device(s)
orig = dev._emit_split
for mode in ("ids", "rows"):
    if mode == "rows":
        dev._emit_split = lambda *a: orig(*a[:10], True, *a[11:])
    for _ in range(3):
        dev.run_join(R, S, k, k)
    torch.cuda.synchronize()
    probe = dev.PhaseProbe()
    for _ in range(5):
        dev.run_join(R, S, k, k, probe=probe)
    torch.cuda.synchronize()
    print(mode, json.dumps({a: round(b / 5 * 1e3, 4) for a, b in probe.durations().items()}))
