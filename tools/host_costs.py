#!/usr/bin/env python
"""Micro-costs of the Python driver's per-join host operations (experiments)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1908_11740_b200 import _native  # noqa: E402
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

d = torch.device("cuda", 0)
torch.cuda.set_device(0)
x = torch.empty(1000, device=d)


def t(name, fn, n=2000):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:40s} {1e6 * (time.perf_counter() - t0) / n:7.2f} us")


t("current_stream(device).cuda_stream", lambda: torch.cuda.current_stream(d).cuda_stream)
t("current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("_C._cuda_getCurrentRawStream(0)", lambda: torch._C._cuda_getCurrentRawStream(0))
t("str(device)", lambda: str(d))
t("tensor.data_ptr()", lambda: x.data_ptr())
t("torch.empty((1000,2), int64, cuda)", lambda: torch.empty((1000, 2), dtype=torch.int64, device=d))
t("buf[:n].view(shape)", lambda: x[:500].view(250, 2))
t("torch.cuda.Event()", lambda: torch.cuda.Event())
lib = _native.load()
h = _native.Header()
t("Header.as_dict()", lambda: h.as_dict())
r, s, k = make_config(1, 0.2)
R, S = dev.to_device(r, d), dev.to_device(s, d)
dev.run_join(R, S, k, k)
dev.run_join(R, S, k, k)
t("run_join cfg1 x0.2 (speculative)", lambda: dev.run_join(R, S, k, k), n=300)
