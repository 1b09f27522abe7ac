"""Host→device copy bandwidth from pinned memory: one stream vs several
streams / chunk sizes (is the e2e join's 800 MB copy at the link's limit?)."""
import torch

N = 800_000_000 // 8
host = torch.empty(N, dtype=torch.float64).pin_memory()
host.fill_(0.5)
dev = torch.empty(N, dtype=torch.float64, device="cuda")
back = torch.empty(N // 20, dtype=torch.float64).pin_memory()


def run(nstreams, chunk_mb, d2h=False):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = chunk_mb * 1_000_000 // 8
    torch.cuda.synchronize()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for st in streams:
        st.wait_event(s0)
    k = 0
    for off in range(0, N, chunk):
        st = streams[k % nstreams]
        with torch.cuda.stream(st):
            dev[off:off + chunk].copy_(host[off:off + chunk], non_blocking=True)
        k += 1
    if d2h:
        with torch.cuda.stream(streams[-1]):
            back.copy_(dev[:N // 20], non_blocking=True)
    for st in streams:
        e = torch.cuda.Event()
        e.record(st)
        torch.cuda.current_stream().wait_event(e)
    e0.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(e0)
    return ms, 800 / ms


for cfg in [(1, 800), (1, 80), (2, 80), (4, 80), (2, 16), (4, 16), (8, 8), (1, 800, True)]:
    best = min(run(*cfg)[0] for _ in range(5))
    print(cfg, f"{best:.2f} ms", f"{800 / best:.1f} GB/s")
