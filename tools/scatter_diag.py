"""Phase split of one config under a library variant (PBSM_LIB_NAME) — for
diagnostic builds whose results are wrong (no parity check)."""
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
for _ in range(3):
    dev.run_join(R, S, k, k)
torch.cuda.synchronize()
probe = dev.PhaseProbe()
for _ in range(5):
    dev.run_join(R, S, k, k, probe=probe)
torch.cuda.synchronize()
print(json.dumps({a: round(b / 5 * 1e3, 4) for a, b in probe.durations().items()}))
