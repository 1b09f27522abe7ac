"""Kernel timeline of one graph-replayed join (CUPTI through torch.profiler):
start offset, duration and stream of every kernel of the step, plus the idle
gaps — shows what overlaps and where the GPU waits.
usage: python tools/timeline.py [config] [row_lo row_hi]"""
import json
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1908_11740_b200 import device as dev  # noqa: E402
from paper_1908_11740_b200 import parallel  # noqa: E402
from paper_1908_11740_b200.synth import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
r, s, k = make_config(cfg, 1.0)
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, k)
if (lo, hi) != (0, k):
    rr = parallel.strip_inputs(r, k, lo, hi)
    ss = rr if s is r else parallel.strip_inputs(s, k, lo, hi)
    r, s = rr, ss
R = dev.to_device(r, "cuda")
S = R if s is r else dev.to_device(s, "cuda")
for _ in range(5):
    dev.run_join(R, S, k, k, row_lo=lo, row_hi=hi, graph=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        dev.run_join(R, S, k, k, row_lo=lo, row_hi=hi, graph=True)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
# the last replay: kernels after the last k_init
starts = [i for i, e in enumerate(ev) if "k_init" in e.name]
ev = ev[starts[-1]:]
t0 = ev[0].time_range.start
end_prev = t0
rows = []
for e in ev:
    name = e.name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    st, en = e.time_range.start - t0, e.time_range.end - t0
    rows.append({"kernel": name[:60], "start_us": round(st, 1), "dur_us": round(en - st, 1),
                 "end_us": round(en, 1), "stream": getattr(e, "stream", None) or e.device_index})
for x in rows:
    print(json.dumps(x))
print(json.dumps({"config": cfg, "rows": [lo, hi], "span_us": rows[-1]["end_us"],
                  "sum_kernel_us": round(sum(x["dur_us"] for x in rows), 1)}))
