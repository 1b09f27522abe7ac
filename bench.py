#!/usr/bin/env python
"""Benchmark of the PBSM filter step (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

One *step* = one complete join (count → plan → scatter → sort+sweep count →
emit, collect-pairs mode) over config C's inputs already resident in HBM;
default C = 2 (BASELINE configs[1]: 10M × 10M MBRs, 2000² grid).  ``value`` is
the whole-job (|R|+|S|) rects/s; pairs/s rides along.  ``e2e`` is the same
metric through the public ``join()`` call with pinned host inputs and the pair
list copied back to host memory every step.  With N > 1 (torchrun) the grid
is split into N tile-row strips (one per rank, weighted by per-row work) and
each rank joins its strip; the per-rank counts are combined by one
all_gather (see paper_1908_11740_b200/parallel.py).

``--impl reference`` times the reference's CPU path (the C restatement in
oracle/, the only place this script executes oracle code besides the
cpu_baseline leg) with all host threads, on a bounded sample of the same
workload, and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "join throughput: (|R|+|S|) rects/sec and result pairs/sec at 1/2/4/8 B200"
UNIT = "rects/s"
ALG_NOTE = ("B_alg = 40(n_R+n_S) + 80(A_R+A_S) + 16P (SURVEY.md §8(d)): MBR+id read once, "
            "tile-list entry written+read once, pair written once")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of CPU work for the cpu_baseline sample")
    ap.add_argument("--traffic-json", default=str(ROOT / "profiles" / "traffic.json"))
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"  # B200_PROFILING.md fallback copy bandwidth


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as exc:  # no NVML: report the gap instead of failing the bench
            self.err = repr(exc)
        return self

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = get_reasons(self.h)
                self.samples.append((time.perf_counter(), float(sm), int(rs)))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        lo, hi = getattr(self, "t_begin", None), getattr(self, "t_end", None)
        if lo is not None and hi is not None:
            inside = [x for x in self.samples if lo <= x[0] <= hi]
            # the step can be shorter than the sampling period: keep the
            # samples nearest the window (warm-up runs the same kernels)
            if len(inside) < 3:
                inside = sorted(self.samples, key=lambda x: min(abs(x[0] - lo), abs(x[0] - hi)))[:5]
            self.samples = inside
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": [],
                    "samples": 0, "note": getattr(self, "err", "no samples")}
        reasons = set()
        for _, _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(x[1] for x in self.samples),
                "sm_max_mhz": float(self.max_mhz), "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU legs
def cpu_sample(cfg: int, budget_s: float, threads: int, probe_f: float = 0.02):
    """A bounded sample of the workload for the CPU: the rectangles overlapping
    a bottom strip of the square (same density as the full job)."""
    import oracle
    from paper_1908_11740_b200.synth import make_config

    r, s, k = make_config(cfg)
    n_total = len(r[0]) + (0 if s is r else len(s[0]))

    def strip(b, f):
        m = b[3] < f  # yl below the strip top
        return tuple(a[m] for a in b)

    frac = 1.0
    # probe on a small strip, then size the sample to the budget
    rp = strip(r, probe_f)
    sp = rp if s is r else strip(s, probe_f)
    t = oracle.join(rp, sp, "2d", k, threads=threads)["total_time"]
    per_frac = max(t / probe_f, 1e-6)
    frac = min(1.0, budget_s / per_frac)
    rs = strip(r, frac) if frac < 1.0 else r
    ss = (rs if s is r else (strip(s, frac) if frac < 1.0 else s))
    n = len(rs[0]) + (0 if s is r else len(ss[0]))
    return rs, ss, k, frac, n, n_total


def run_cpu(cfg, threads, rs, ss, k):
    import oracle

    res = oracle.join(rs, ss, "2d", k, threads=threads)
    return res


def physical_cores():
    try:
        import psutil
        return psutil.cpu_count(logical=False) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    rs, ss, k, frac, n, n_total = cpu_sample(args.config, budget, threads, probe_f=0.1)
    for _ in range(args.warmup):
        run_cpu(args.config, threads, rs, ss, k)
    t0 = time.perf_counter()
    pairs = 0
    for _ in range(args.steps):
        res = run_cpu(args.config, threads, rs, ss, k)
        pairs = res["count"]
    dt = (time.perf_counter() - t0) / args.steps
    value = n / dt
    sample = (f"cfg{args.config} rectangles with yl < {frac:.4f} (a bottom strip, "
              f"{n} of {n_total} rects, {pairs} pairs), oracle C port of the reference path, "
              f"{threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "pairs_per_s": pairs / dt,
        "config": {"workload": f"cfg{args.config}", "sample_fraction": frac},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def h2d_floor(rh, sh, e2e_s: float) -> dict:
    """The e2e join's floor: the same pinned input columns copied host→device
    alone (one stream, back to back, CUDA events; best of 3).  ``frac`` =
    that copy time ÷ the e2e step time (1.0 = the join adds nothing to the
    PCIe transfer of its inputs)."""
    import torch

    cols = [c for b in (rh, sh) if b is not None for c in (b.ids, b.xl, b.xu, b.yl, b.yu)]
    host = [torch.from_numpy(c) for c in cols]
    dev = [torch.empty_like(h, device="cuda") for h in host]
    st = torch.cuda.Stream()
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            for d_, h_ in zip(dev, host):
                d_.copy_(h_, non_blocking=True)
            e1.record(st)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    nbytes = sum(h.numel() * h.element_size() for h in host)
    del dev
    return {"h2d_GBps": nbytes / best / 1e9, "h2d_ms": best * 1e3, "frac": best / e2e_s,
            "note": "input columns copied alone from the same pinned buffers"}


def count_launches(h: dict, dev, n_r: int, n_s: int) -> int:
    """Our kernels per join step (see device.run_join / pbsm.cu host glue)."""
    n = 1            # k_init
    n += 2           # k_count R, S
    n += 3           # k_plan_reduce, k_plan_partials, k_plan_apply
    n += 2           # k_scatter R, S
    for total, m in ((h["list_r"], n_r), (h["list_s"], n_s)):
        # binned scatter: 3 scan kernels + k_bin_copy
        n += 4 if dev._binned(total, m, None) else 0
    # k_join_nested (with the write guard fused in) or a stand-alone k_guard
    n += 1
    n += 1 if h["chunks_sorted"] + h["n_items"] > 0 else 0   # k_join (sorted / large units)
    n += 1           # k_publish_header (the final header read)
    return n


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_1908_11740_b200 import JoinConfig, PartitionLayout, RectBatch
    from paper_1908_11740_b200 import device as dev
    from paper_1908_11740_b200 import engine, parallel
    from paper_1908_11740_b200.synth import CONFIGS, make_config

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with "
                                       f"{args.gpus} processes"}))
            return 1
    # test hook (tools/multirank_smoke.sh): PBSM_BENCH_SHARED_GPU=1 runs every
    # rank on cuda:0 with gloo collectives — exercises the multi-rank host
    # logic on a one-GPU box (no kernel waits on another rank); the numbers of
    # such a run are not a measurement
    shared = os.environ.get("PBSM_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)

    spec = CONFIGS[args.config]
    r, s, k = make_config(args.config)
    n_r, n_s = len(r[0]), len(s[0])
    self_join = s is r
    # strip plan (host side, before the timed region)
    plan = parallel.plan_strips(r, s, k, world)
    row_lo, row_hi = plan[rank], plan[rank + 1]
    rr = parallel.strip_inputs(r, k, row_lo, row_hi)
    ss = rr if self_join else parallel.strip_inputs(s, k, row_lo, row_hi)
    rd = dev.to_device(rr, device)
    sd = rd if self_join else dev.to_device(ss, device)
    torch.cuda.synchronize()

    def step(probe=None):
        res = dev.run_join(rd, sd, k, k, collect=True, row_lo=row_lo, row_hi=row_hi,
                           probe=probe)
        if world > 1:
            # the one collective: all_gather {pairs, A_R, A_S} → global pair offset
            res.header["exchange"] = parallel.exchange_counts(
                res.count, res.header["a_r"], res.header["a_s"], device=device)
        return res

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local).__enter__()  # running through warm-up: no start-up gap
    for _ in range(max(3, args.warmup)):
        res = step()
    barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    barrier()
    clocks.t_begin = time.perf_counter()
    start.record()
    for _ in range(args.steps):
        res = step()
    end.record()
    barrier()
    clocks.t_end = time.perf_counter()
    t_local = start.elapsed_time(end) / 1e3
    # per-phase device times: the same K steps again, outside the timed
    # region (the phase events add host work between the launches)
    probe = dev.PhaseProbe()
    for _ in range(args.steps):
        step(probe)
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    t = t_local
    local_pairs = res.count
    totals = parallel.combine_counts(res.count, res.header["a_r"], res.header["a_s"], t_local,
                                     world, device=device)
    t = totals["t_max"]
    P = totals["pairs"]
    A_R, A_S = totals["a_r"], totals["a_s"]
    step_s = t / args.steps
    value = (n_r + n_s) / step_s
    phases = {k_: v / args.steps for k_, v in probe.durations().items() if k_ != "start"}

    hbm, peak_kind = peaks()
    B_alg = 40 * (n_r + n_s) + 80 * (A_R + A_S) + 16 * P
    step_gbs = B_alg / step_s / 1e9
    # dominant kernel: the longest device phase
    dev_phases = {k_: v for k_, v in phases.items() if not k_.startswith("header")}
    dom = max(dev_phases, key=dev_phases.get)
    h = res.header
    # algorithmic bytes of each phase, per SURVEY §8(d)'s per-unit figures
    n_in = len(rr[0]) + len(ss[0])   # both inputs are partitioned (engine.py:231-232)
    lists = h["list_r"] + h["list_s"]
    dom_bytes = {
        "count": 32 * n_in,                           # every MBR read once
        "scatter": 40 * n_in + 40 * lists,            # MBR+id read, entry written
        "join": 40 * lists + 16 * local_pairs,        # entry read, pair written
        "plan": 4 * 6 * (k * (row_hi - row_lo)),
        "bin": 80 * n_in,
        "init": 8 * k * (row_hi - row_lo),
    }[dom]
    # the dominant phase runs one launch per input (count, scatter) or the
    # nested + sorted/large join launches; report per launch of its kernel
    n_launch = {"count": 2, "scatter": 2, "bin": 2}.get(dom, 1)
    dom_bytes //= n_launch
    dom_time = dev_phases[dom] / n_launch
    dom_gbs = dom_bytes / dom_time / 1e9
    traffic = None
    tp = Path(args.traffic_json)
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(f"cfg{args.config}", {}).get(dom)
        except Exception:
            traffic = None

    # e2e through the public API: pinned host inputs → join() → pairs on host
    e2e = None
    if not args.no_e2e and world == 1:
        import torch as _t

        def pinned(b):
            out = []
            for a in b:
                t_ = _t.empty(a.shape, dtype=_t.from_numpy(a[:1]).dtype, pin_memory=True)
                t_.numpy()[:] = a
                out.append(t_.numpy())
            return RectBatch(*out)

        Rh = pinned(r)
        Sh = Rh if self_join else pinned(s)
        cfgj = JoinConfig(PartitionLayout("2d", k), sink_mode="collect-pairs")
        rep = engine.join(Rh, Sh, cfgj)  # warm
        ts = []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = engine.join(Rh, Sh, cfgj)
            ts.append(time.perf_counter() - t0)
        e2e_t = statistics.median(ts)
        h2d = 40 * (n_r + (0 if self_join else n_s))
        e2e = {"value": (n_r + n_s) / e2e_t, "unit": UNIT,
               "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 16 * rep.result_count, "ms_per_step": e2e_t * 1e3,
               "api": "paper_1908_11740_b200.join(RectBatch, RectBatch, JoinConfig("
                      "PartitionLayout('2d', K), sink_mode='collect-pairs'))",
               "link": h2d_floor(Rh, None if self_join else Sh, e2e_t)}
    elif not args.no_e2e:
        # N ranks: each rank's strip (split on the host beforehand — the
        # distribution step) from pinned host memory through the public strip
        # API: H2D, join, count exchange, its pair shard back to the host
        import torch as _t

        def pinned_cols(b):
            out = []
            for a in b:
                t_ = _t.empty(a.shape, dtype=_t.from_numpy(a[:1]).dtype, pin_memory=True)
                t_.numpy()[:] = a
                out.append(t_.numpy())
            return tuple(out)

        rh = pinned_cols(rr)
        sh = rh if self_join else pinned_cols(ss)
        parallel.strip_join(rh, sh, k, row_lo, row_hi, device)  # warm
        ts = []
        for _ in range(args.e2e_steps):
            barrier()
            t0 = time.perf_counter()
            sres, sex = parallel.strip_join(rh, sh, k, row_lo, row_hi, device)
            host_pairs = torch.empty(tuple(sres.pairs.shape), dtype=torch.int64, pin_memory=True)
            host_pairs.copy_(sres.pairs)
            ts.append(time.perf_counter() - t0)
        tl = torch.tensor([statistics.median(ts), 40.0 * (len(rh[0]) + (0 if self_join
                                                                          else len(sh[0])))],
                          dtype=torch.float64, device=device)
        tmax = tl[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tl, op=dist.ReduceOp.SUM)
        e2e_t = float(tmax.item())
        e2e = {"value": (n_r + n_s) / e2e_t, "unit": UNIT,
               "h2d_bytes_per_step": int(tl[1].item()),
               "d2h_bytes_per_step": 16 * int(sex["pairs"]), "ms_per_step": e2e_t * 1e3,
               "api": "paper_1908_11740_b200.parallel.strip_join(strip R, strip S, K, "
                      "row_lo, row_hi) per rank (host strip split outside the timed region)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rs_, ss_, k_, frac, n_smp, n_tot = cpu_sample(args.config, args.cpu_budget, threads)
        t0 = time.perf_counter()
        cres = run_cpu(args.config, threads, rs_, ss_, k_)
        ct = time.perf_counter() - t0
        cpu = {"value": n_smp / ct, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"cfg{args.config} rectangles with yl < {frac:.4f} ({n_smp} of "
                         f"{n_tot} rects, {cres['count']} pairs); oracle/pbsm_oracle.c "
                         f"(C restatement of the reference path), {threads} threads, 1 run",
               "pairs_per_s": cres["count"] / ct}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    launches = count_launches(res.header, dev, len(rr[0]), len(ss[0])) * args.steps
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SURVEY.md §8(d) generators; TIGER/OSM data unavailable)",
        "config": {"workload": f"cfg{args.config}", "n_r": n_r, "n_s": n_s, "grid": f"{k}x{k}",
                   "self_join": self_join, "sink_mode": "collect-pairs",
                   "parallelism": f"strips{world}",
                   "l2": f"no flush: inputs {40 * (n_r + n_s) / 1e6:.0f} MB + tile lists "
                         f"{40 * (A_R + A_S) / 1e6:.0f} MB > 126 MB L2"},
        "pairs": P, "pairs_per_s": P / step_s, "a_r": A_R, "a_s": A_S,
        "roofline": {"bound": "hbm", "kernel": {"scatter": "k_scatter", "count": "k_count",
                                                 "join": "k_join_nested+k_join",
                                                 "bin": "k_bin_copy"}.get(dom, dom),
                     "phase": dom, "achieved": dom_gbs, "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": dom_gbs / hbm,
                     "traffic": traffic, "alg_bytes_per_launch": dom_bytes,
                     "launches_per_step": n_launch, "launch_ms": dom_time * 1e3,
                     "timing": "phase span on the launch stream (CUDA events) / launches: "
                               "R's and S's count/scatter launches run concurrently on two "
                               "streams, so this is the phase's aggregate rate"},
        "step_roofline": {"alg_bytes": B_alg, "achieved": step_gbs, "peak": hbm * world,
                          "frac": step_gbs / (hbm * world), "unit": "GB/s", "formula": ALG_NOTE},
        "phases_ms": {k_: v * 1e3 for k_, v in phases.items()},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
