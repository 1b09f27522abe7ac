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

``--impl reference`` times the reference's CPU path on the SAME full config
every step (the C restatement in oracle/ with all host threads — the only
place this script executes oracle code) and prints the same JSON line with
"impl": "reference".  The GPU arm's ``cpu_baseline`` times the reference's
own compiled ``sweepjoin.join`` (installed into baseline/_ref by
oracle/build_ref.sh) on the full config.  Both arms gate their output on the
reference's full-size truth (``parity``: count, A_R, A_S and the sha256 of the
sorted pair list, tests/golden/full_truth.json); a mismatch exits 1.
"""

from __future__ import annotations

import argparse
import datetime
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
    ap.add_argument("--cpu-variants", default="x1,xN",
                    help="cpu_baseline runs of the reference join: axis x|a(daptive) + "
                         "threads (N = physical cores), e.g. x1,xN,a1,aN")
    ap.add_argument("--sub-configs", default="5,3,4",
                    help="other BASELINE configs timed in the same run (N=1), '' or none for none")
    ap.add_argument("--sub-steps", type=int, default=5)
    ap.add_argument("--no-parity", action="store_true")
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


# ---------------------------------------------------------------- parity
TRUTH = ROOT / "tests" / "golden" / "full_truth.json"


def truth_for(cfg: int):
    """Full-size truth computed by the reference itself
    (tests/golden/make_full_truth.py): count, A_R, A_S, sha256 of the sorted list."""
    if not TRUTH.exists():
        return None
    return json.loads(TRUTH.read_text()).get(f"cfg{cfg}")


def sorted_sha256_host(pairs: np.ndarray) -> str:
    import hashlib

    p = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if len(p):
        p = p[np.lexsort((p[:, 1], p[:, 0]))]
    return hashlib.sha256(np.ascontiguousarray(p, dtype="<i8").tobytes()).hexdigest()


def sorted_sha256_device(pairs) -> str:
    """sha256 of the lexicographically sorted pair list (sorted on the device,
    hashed on the host) — the parity form of the unordered list."""
    import hashlib

    from paper_1908_11740_b200 import parallel

    p = parallel.canonical_pairs(pairs.contiguous()).cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(p, dtype="<i8").tobytes()).hexdigest()


def parity_record(cfg: int, count: int, a_r: int, a_s: int, digest: str) -> dict:
    t = truth_for(cfg)
    if t is None:
        return {"match": None, "sha256": digest, "note": "no committed truth"}
    ok = (count == t["count"] and a_r == t["a_r"] and a_s == t["a_s"]
          and digest == t["pairs_sha256"])
    return {"match": bool(ok), "sha256": digest[:16], "count": count,
            "truth": "tests/golden/full_truth.json (reference sweepjoin.join, threads=1, "
                     "full size)"}


# ---------------------------------------------------------------- CPU legs
def physical_cores():
    try:
        import psutil
        return psutil.cpu_count(logical=False) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def import_reference():
    """The unmodified reference package installed by oracle/build_ref.sh into
    baseline/_ref (git-ignored; travels to the GPU box), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "sweepjoin").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import sweepjoin
        if "compiled" not in sweepjoin.available_backends():
            return None
        return sweepjoin
    except Exception:
        return None


def reference_cpu_baseline(cfg: int, variants: str) -> dict | None:
    """BASELINE.md §2's CPU baseline: the reference's own compiled backend,
    sweepjoin.join(R, S, JoinConfig(PartitionLayout("2d", K), axis_policy=...,
    sink_mode="collect-pairs", threads=...)) on the FULL config, one run per
    variant, best reported (JoinReport.total_time, inputs already in memory)."""
    sj = import_reference()
    if sj is None:
        return None
    from paper_1908_11740_b200.synth import make_config

    r, s, k = make_config(cfg)
    R = sj.RectBatch(*r)
    S = R if s is r else sj.RectBatch(*s)
    n = len(r[0]) + len(s[0])
    cores = physical_cores()
    runs = []
    for v in variants.split(","):
        v = v.strip()
        if not v:
            continue
        axis = {"x": "x", "a": "adaptive"}[v[0]]
        threads = cores if v[1:] == "N" else int(v[1:])
        rep = sj.join(R, S, sj.JoinConfig(sj.PartitionLayout("2d", k), axis_policy=axis,
                                          sink_mode="collect-pairs", threads=threads))
        runs.append({"axis_policy": axis, "threads": threads, "total_time_s": rep.total_time,
                     "pairs": int(rep.result_count)})
        del rep
    if not runs:
        return None
    best = min(runs, key=lambda x: x["total_time_s"])
    return {"value": n / best["total_time_s"], "unit": UNIT, "cores": best["threads"],
            "kind": "reference",
            "sample": f"full cfg{cfg} ({n} rects, {best['pairs']} pairs): reference sweepjoin "
                      f"{getattr(sj, '__version__', '0.1.0')} compiled backend (baseline/_ref, "
                      f"oracle/build_ref.sh), best of {len(runs)} variant(s)",
            "pairs_per_s": best["pairs"] / best["total_time_s"], "variants": runs,
            "host_cores_physical": cores, "host_cpu": host_cpu()}


def port_cpu_baseline(cfg: int) -> dict:
    """Fallback when baseline/_ref is absent: the C port, full config, all threads."""
    import oracle
    from paper_1908_11740_b200.synth import make_config

    r, s, k = make_config(cfg)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    res = oracle.join(r, s, "2d", k, threads=threads)
    dt = time.perf_counter() - t0
    n = len(r[0]) + len(s[0])
    return {"value": n / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"full cfg{cfg} ({n} rects, {res['count']} pairs), oracle/pbsm_oracle.c "
                      f"(C restatement of the reference path), {threads} threads, 1 run",
            "pairs_per_s": res["count"] / dt, "host_cpu": host_cpu()}


def host_cpu() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_arm(args):
    """``--impl reference``: the reference CPU path on the arm's own config —
    the FULL config every step (no sample), through the C restatement of the
    reference's compiled path (oracle/pbsm_oracle.c, kind "port") with every
    host thread (the reference's own join() takes 34 s per cfg2 step at its
    best setting; bench.py's cpu_baseline leg times it)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from paper_1908_11740_b200.synth import make_config

    threads = os.cpu_count() or 1
    r, s, k = make_config(args.config)
    n = len(r[0]) + len(s[0])
    res = None
    for _ in range(args.warmup):
        res = oracle.join(r, s, "2d", k, threads=threads)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = oracle.join(r, s, "2d", k, threads=threads)
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / len(ts)
    value = n / dt
    parity = parity_record(args.config, res["count"], res["a_r"], res["a_s"],
                           sorted_sha256_host(res["pairs"]))
    sample = (f"full cfg{args.config} every step ({n} rects, {res['count']} pairs), "
              f"oracle/pbsm_oracle.c (C restatement of the reference's compiled path), "
              f"{threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "pairs_per_s": res["count"] / dt,
        "config": {"workload": f"cfg{args.config}", "same_config": True, "n_r": len(r[0]),
                   "n_s": len(s[0]), "grid": f"{k}x{k}", "sink_mode": "collect-pairs"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "host_cpu": host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": parity,
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
            # a stuck collective must fail the run, not hang the box
            os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
            dist.init_process_group("nccl", device_id=device,
                                    timeout=datetime.timedelta(seconds=120))

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
        # (repeated joins of the same resident inputs replay one CUDA graph;
        # the phase-probe pass runs the same launches eagerly)
        # world > 1: the join's one collective (all_gather {pairs, A_R, A_S} →
        # global pair offset) — inside the graph, from the device header
        res = dev.run_join(rd, sd, k, k, collect=True, row_lo=row_lo, row_hi=row_hi,
                           probe=probe, graph=True, exchange=world > 1)
        return res

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # cold latency: the first join of this shape in the process (synchronous
    # plan-header read, first allocations of the tile lists and scratch)
    barrier()
    t0 = time.perf_counter()
    res = step()
    torch.cuda.synchronize()
    cold_ms = (time.perf_counter() - t0) * 1e3
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
    step(dev.PhaseProbe())  # (the eager path's own buffers, allocated untimed)
    probe = dev.PhaseProbe()
    for _ in range(args.steps):
        step(probe)
    torch.cuda.synchronize()
    clocks.__exit__(None, None, None)
    # parity gate: the last timed step's pair list, sorted on the device and
    # hashed, against the reference's full-size truth
    parity = None
    if not args.no_parity:
        allp = res.pairs
        if world > 1:
            ex = parallel.exchange_counts(res.count, res.header["a_r"], res.header["a_s"],
                                          device=device)
            allp = parallel.gather_pairs(res.pairs, ex, dst=0)
        if rank == 0:
            ex0 = parallel.exchange_counts(res.count, res.header["a_r"], res.header["a_s"],
                                           device=device) if world == 1 else ex
            parity = parity_record(args.config, ex0["pairs"], ex0["a_r"], ex0["a_s"],
                                   sorted_sha256_device(allp))
        del allp
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
    once = self_join and dev.SELF_ONCE  # one array, partitioned once: its bytes move once
    if once:
        B_alg = 40 * n_r + 80 * A_R + 16 * P
    step_gbs = B_alg / step_s / 1e9
    # dominant kernel: the longest device phase
    dev_phases = {k_: v for k_, v in phases.items()
                  if not k_.startswith("header") and k_ not in ("alloc", "start")}
    dom = max(dev_phases, key=dev_phases.get)
    h = res.header
    # algorithmic bytes of each phase, per SURVEY §8(d)'s per-unit figures
    n_in = len(rr[0]) + len(ss[0])   # both inputs are partitioned (engine.py:231-232)
    lists = h["list_r"] + h["list_s"]
    if once:  # ... unless they are one array: one count, one scatter, one list
        n_in, lists = len(rr[0]), h["list_r"]
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
    n_launch = 1 if once else {"count": 2, "scatter": 2, "bin": 2}.get(dom, 1)
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

    subs = {}
    sub_list = [x.strip() for x in args.sub_configs.split(",")
                if x.strip() and x.strip().lower() != "none"]
    if rank == 0 and world == 1 and sub_list:
        del rd, sd
        dev.release_buffers()
        torch.cuda.empty_cache()
        for c in [int(x) for x in sub_list]:
            if c == args.config:
                continue
            subs[f"cfg{c}"] = time_sub_config(c, args.sub_steps, device, hbm, args.no_parity)
            dev.release_buffers()
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = reference_cpu_baseline(args.config, args.cpu_variants)
        if cpu is None:
            cpu = port_cpu_baseline(args.config)

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
        "cold_first_join_ms": cold_ms,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": parity,
        "sub_configs": subs,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    bad = [name for name, v in [(f"cfg{args.config}", {"parity": parity})] + list(subs.items())
           if (v.get("parity") or {}).get("match") is False]
    if bad:
        print(f"PARITY MISMATCH against tests/golden/full_truth.json: {bad}", file=sys.stderr)
        return 1
    return 0


def time_sub_config(cfg: int, steps: int, device, hbm: float, no_parity: bool) -> dict:
    """Another BASELINE config in the same run: device-resident inputs, 2
    warm-up joins, ``steps`` timed joins (CUDA events), the step roofline and
    the parity hash of the last join."""
    import torch

    from paper_1908_11740_b200 import device as dev
    from paper_1908_11740_b200.synth import make_config

    r, s, k = make_config(cfg)
    n = len(r[0]) + len(s[0])
    rd = dev.to_device(r, device)
    sd = rd if s is r else dev.to_device(s, device)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = dev.run_join(rd, sd, k, k)
    torch.cuda.synchronize()
    cold = (time.perf_counter() - t0) * 1e3
    for _ in range(3):
        res = dev.run_join(rd, sd, k, k, graph=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        res = dev.run_join(rd, sd, k, k, graph=True)
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / steps
    h = res.header
    b_alg = 40 * n + 80 * (h["a_r"] + h["a_s"]) + 16 * res.count
    once = s is r and dev.SELF_ONCE
    if once:  # a self-join partitions its one array once: those bytes move once
        b_alg = 40 * len(r[0]) + 80 * h["a_r"] + 16 * res.count
    out = {"ms_per_step": dt * 1e3, "value": n / dt, "unit": UNIT, "pairs": res.count,
           "a_r": h["a_r"], "a_s": h["a_s"], "steps": steps, "cold_first_join_ms": cold,
           "step_roofline": {"alg_bytes": b_alg, "achieved": b_alg / dt / 1e9, "peak": hbm,
                             "frac": b_alg / dt / 1e9 / hbm, "unit": "GB/s"}}
    if once:
        out["self_join"] = ("partitioned once (R is S): B_alg = 40 n_R + 80 A_R + 16 P; the "
                            "reference partitions the array twice (engine.py:231-232)")
    if not no_parity:
        out["parity"] = parity_record(cfg, res.count, h["a_r"], h["a_s"],
                                      sorted_sha256_device(res.pairs))
    del res, rd, sd
    dev.release_buffers()  # (this config's lists, scratch and graph)
    return out


if __name__ == "__main__":
    sys.exit(main())
