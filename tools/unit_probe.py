"""Time the unit pipeline against the tile-list pipeline on one config
(device-resident inputs, CUDA events, phase split from PhaseProbe)."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

cfgs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2").split(",")]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for cfg in cfgs:
    r, s, k = make_config(cfg)
    R = dev.to_device(r)
    S = R if s is r else dev.to_device(s)
    torch.cuda.synchronize()
    out = {"cfg": cfg}
    for pipe in ("units", "tiles"):
        for _ in range(3):
            res = dev.run_join(R, S, k, k, pipeline=pipe)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            res = dev.run_join(R, S, k, k, pipeline=pipe)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        probe = dev.PhaseProbe()
        for _ in range(steps):
            dev.run_join(R, S, k, k, pipeline=pipe, probe=probe)
        torch.cuda.synchronize()
        ph = {a: round(b / steps * 1e3, 4) for a, b in probe.durations().items()}
        out[pipe] = {"ms": round(ms, 4), "count": res.count, "phases_ms": ph,
                     "header": {a: b for a, b in res.header.items() if isinstance(b, int)}}
        dev.release_buffers()
    print(json.dumps(out), flush=True)
