"""cfg join phase vs the large-tile threshold sweep_min (brute force below,
sort + forward scan above)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
r, s, k = make_config(cfg)
R = dev.to_device(r)
S = R if s is r else dev.to_device(s)
for sm in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "67108864,4194304,1048576,262144,65536").split(",")]:
    for _ in range(3):
        res = dev.run_join(R, S, k, k, sweep_min=sm)
    torch.cuda.synchronize()
    probe = dev.PhaseProbe()
    for _ in range(5):
        res = dev.run_join(R, S, k, k, sweep_min=sm, probe=probe)
    torch.cuda.synchronize()
    ph = {a: round(b / 5 * 1e3, 3) for a, b in probe.durations().items()}
    print(json.dumps({"cfg": cfg, "sweep_min": sm, "pairs": res.count, "max_huge": res.header["max_huge"],
                      "phases_ms": ph}), flush=True)
    dev.release_buffers()
