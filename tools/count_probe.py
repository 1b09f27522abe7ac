#!/usr/bin/env python
"""Time pbsm_init + pbsm_count (both inputs) alone with CUDA events (experiments;
works with diagnostic builds whose later phases would fail).  PBSM_LIB_NAME
selects the library variant.  usage: count_probe.py [--config 2] [--reps 10]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1908_11740_b200 import _native
from paper_1908_11740_b200 import device as dev
from paper_1908_11740_b200.synth import CONFIGS, make_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
r, s, k = make_config(a.config, 1.0)
R = dev.to_device(r, "cuda")
S = R if s is r else dev.to_device(s, "cuda")
lib = _native.load()
ws = dev._workspace(lib, torch.device("cuda"), k, k, 0, k)
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
t_init = t_cnt = 0.0
for it in range(a.reps + 2):
    ev[0].record()
    lib.pbsm_init(ws.data_ptr(), k, k, 0, k, st)
    ev[1].record()
    for side, b in ((0, R), (1, S)):
        lib.pbsm_count(b.xl.data_ptr(), b.xu.data_ptr(), b.yl.data_ptr(), b.yu.data_ptr(), len(b),
                       side, ws.data_ptr(), k, k, 0, k, st)
    ev[2].record()
    ev[2].synchronize()
    if it >= 2:
        t_init += ev[0].elapsed_time(ev[1])
        t_cnt += ev[1].elapsed_time(ev[2])
print(f"{CONFIGS[a.config].name} init {t_init / a.reps:.3f} ms count {t_cnt / a.reps:.3f} ms")
