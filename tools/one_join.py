"""N joins of one config through run_join (for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pipe = sys.argv[3] if len(sys.argv) > 3 else None
r, s, k = make_config(cfg)
R = dev.to_device(r)
S = R if s is r else dev.to_device(s)
for _ in range(reps):
    res = dev.run_join(R, S, k, k, pipeline=pipe)
torch.cuda.synchronize()
print(cfg, res.count)
