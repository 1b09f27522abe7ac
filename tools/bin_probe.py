"""Phase split of the binned pipeline (row-band copy + banded scatter) vs the
direct scatter on one config (library variant via PBSM_LIB_NAME)."""
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
out = {"cfg": cfg}
for name, bb in (("direct", None), ("binned", 0)):
    for _ in range(3):
        res = dev.run_join(R, S, k, k, bin_bytes=bb)
    torch.cuda.synchronize()
    probe = dev.PhaseProbe()
    for _ in range(5):
        res = dev.run_join(R, S, k, k, bin_bytes=bb, probe=probe)
    torch.cuda.synchronize()
    out[name] = {a: round(b / 5 * 1e3, 4) for a, b in probe.durations().items()}
    out[name]["pairs"] = res.count
print(json.dumps(out))
