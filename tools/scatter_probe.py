#!/usr/bin/env python
"""Time pbsm_scatter (both inputs) alone with CUDA events, re-running
init/count/plan before each repetition (experiments: works with diagnostic
builds whose guard would fail).  PBSM_LIB_NAME selects the library variant.
usage: scatter_probe.py [--config 2] [--reps 10]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import _native  # noqa: E402
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200.synth import CONFIGS, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
r, s, k = make_config(a.config, 1.0)
R = dev.to_device(r, "cuda")
S = R if s is r else dev.to_device(s, "cuda")
lib = _native.load()
ws = dev._workspace(lib, torch.device("cuda"), k, k, 0, k)
wsp = ws.data_ptr()
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
lists = None
t_c = t_s = 0.0
for it in range(a.reps + 2):
    ev[0].record()
    lib.pbsm_init(wsp, k, k, 0, k, st)
    for side, b in ((0, R), (1, S)):
        lib.pbsm_count(b.xl.data_ptr(), b.xu.data_ptr(), b.yl.data_ptr(), b.yu.data_ptr(), len(b),
                       side, wsp, k, k, 0, k, st)
    lib.pbsm_plan(wsp, k, k, 0, k, -1, -1, st)
    h = _native.Header()
    lib.pbsm_read_header(wsp, h, st)
    if lists is None:
        lists = [torch.empty((max(h.list_r, 1), 8), dtype=torch.int64, device="cuda"),
                 torch.empty((max(h.list_s, 1), 8), dtype=torch.int64, device="cuda")]
    ev[1].record()
    for side, b, tot in ((0, R, h.list_r), (1, S, h.list_s)):
        lib.pbsm_scatter(b.ids.data_ptr(), b.xl.data_ptr(), b.xu.data_ptr(), b.yl.data_ptr(),
                         b.yu.data_ptr(), len(b), side, wsp, k, k, 0, k,
                         lists[side].data_ptr(), tot, st)
    ev[2].record()
    ev[2].synchronize()
    if it >= 2:
        t_c += ev[0].elapsed_time(ev[1])
        t_s += ev[1].elapsed_time(ev[2])
print(f"{CONFIGS[a.config].name} init+count+plan {t_c / a.reps:.3f} ms scatter {t_s / a.reps:.3f} ms")
