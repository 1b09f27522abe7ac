import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_1908_11740_b200 import JoinConfig, PartitionLayout, RectBatch, join
from paper_1908_11740_b200 import device as dev
from paper_1908_11740_b200.synth import make_config
r, s, k = make_config(2)
def pinned(b):
    out=[]
    for a in b:
        t=torch.empty(a.shape, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True); t.numpy()[:]=a; out.append(t.numpy())
    return RectBatch(*out)
R, S = pinned(r), pinned(s)
cfg = JoinConfig(PartitionLayout("2d", k), sink_mode="collect-pairs")
join(R, S, cfg)
for _ in range(3):
    torch.cuda.synchronize(); t0=time.perf_counter()
    rd = dev.to_device(R); sd = dev.to_device(S); torch.cuda.synchronize(); t1=time.perf_counter()
    res = dev.run_join(rd, sd, k, k); torch.cuda.synchronize(); t2=time.perf_counter()
    p = res.pairs.cpu().numpy(); t3=time.perf_counter()
    rep = join(R, S, cfg); t4=time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.1f} join {1e3*(t2-t1):.1f} d2h {1e3*(t3-t2):.1f} | join() total {1e3*(t4-t3):.1f} ms; pinned? {torch.from_numpy(R.xl).is_pinned()}")
