"""Host-side timeline of one end-to-end join() (cfg2, pinned inputs): when
each stage is entered / returns, relative to the join() call — where the
~0.4 ms between the PCIe floor and the e2e step goes.
usage: python tools/e2e_timeline.py [--config 2]"""
import argparse
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import JoinConfig, PartitionLayout, RectBatch, engine  # noqa: E402
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
r, s, k = make_config(a.config)


def pinned(b):
    out = []
    for x in b:
        t = torch.empty(x.shape, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True)
        t.numpy()[:] = x
        out.append(t.numpy())
    return RectBatch(*out)


R = pinned(r)
S = R if s is r else pinned(s)
cfg = JoinConfig(PartitionLayout("2d", k), sink_mode="collect-pairs")
marks = {}


def wrap(name, fn):
    def w(*args, **kw):
        marks.setdefault(name + ">", []).append(time.perf_counter() - T0[0])
        out = fn(*args, **kw)
        marks.setdefault(name + "<", []).append(time.perf_counter() - T0[0])
        return out
    return w


T0 = [0.0]
dev.to_device_pipelined = wrap("to_device", dev.to_device_pipelined)
dev.run_join = wrap("run_join", dev.run_join)
dev.staged_pairs_to_host = wrap("staged", dev.staged_pairs_to_host)
engine.dev = dev
for i in range(8):
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    engine.join(R, S, cfg)
    marks.setdefault("end", []).append(time.perf_counter() - T0[0])
for kk, v in marks.items():
    print(f"{kk:12s} {statistics.median(v[2:]) * 1e3:8.3f} ms")
