"""Command-line front end: ``python -m paper_1908_11740_b200 join|bench``.

The reference CLI's ``join`` and ``bench`` subcommands (cli.py:124-193 in
/root/reference/pkg/src/sweepjoin) over the B200 path: same flags where they
apply, same text / CSV output, inputs in CSV or SJB1 (SJB1 is unpacked on
the GPU, ``io.load_dataset_device``).  ``--backend`` accepts only ``cuda``;
``--verify`` is not offered (the checker lives in the test suite).
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from . import engine
from . import io as pio
from .errors import InvalidStatisticsError, SweepJoinError
from .partition import DEFAULT_K_MAX, PartitionLayout, recommend_k

CSV_HEADER = "layout,k,axis,threads,rep,partition_s,join_s,total_s,result_count"
AUTO_K_MAX_2D = 2048


def _load(path):
    batch, stats = pio.load_dataset(path)
    return batch, stats


def _load_pair(left, right):
    a, sa = _load(left)
    b, sb = _load(right)
    if len(a) and len(b):
        xmin, ymin, xmax, ymax = pio.union_bbox(a, b)
        if xmin < 0.0 or ymin < 0.0 or xmax > 1.0 or ymax > 1.0:
            print("note: data outside the unit square; normalizing both inputs "
                  "by their combined bounding box", file=sys.stderr)
            a, b = pio.normalize_pair(a, b)
            sa, sb = pio.compute_stats(a), pio.compute_stats(b)
    return a, b, sa, sb


def _auto_k(kind, sa, sb, epsilon):
    n = sa.cardinality + sb.cardinality
    if epsilon is not None:
        avg = epsilon
    elif n == 0:
        avg = 0.0
    else:
        ax = (sa.cardinality * sa.avg_x_extent + sb.cardinality * sb.avg_x_extent) / n
        ay = (sa.cardinality * sa.avg_y_extent + sb.cardinality * sb.avg_y_extent) / n
        avg = ax if kind == "1d" else (ax + ay) / 2.0
    k_max = AUTO_K_MAX_2D if kind == "2d" else DEFAULT_K_MAX
    try:
        return recommend_k(avg, kind, k_max=k_max)
    except InvalidStatisticsError:
        print(f"warning: zero average extent (point data); capping K at {k_max}",
              file=sys.stderr)
        return k_max


def _resolve_k(value, kind, sa, sb, epsilon):
    if value == "auto":
        return _auto_k(kind, sa, sb, epsilon)
    k = int(value)
    if k < 1:
        raise SweepJoinError(f"k must be >= 1, got {k}")
    return k


def _run(a, b, cfg, epsilon):
    if epsilon is not None:
        return engine.epsilon_distance_join(a, b, epsilon, cfg)
    return engine.join(a, b, cfg)


def _csv_row(layout, axis, threads, rep, rep_):
    return (f"{layout.kind},{layout.k},{axis},{threads},{rep},{rep_.partition_time:.6f},"
            f"{rep_.sort_time + rep_.join_time:.6f},{rep_.total_time:.6f},{rep_.result_count}")


def cmd_join(args) -> int:
    a, b, sa, sb = _load_pair(args.left, args.right)
    k = _resolve_k(args.k, args.layout, sa, sb, args.epsilon)
    layout = PartitionLayout(args.layout, k)
    axis = args.axis or ("auto" if args.layout == "1d" else "adaptive")
    cfg = engine.JoinConfig(layout=layout, axis_policy=axis, threads=args.threads,
                            sink_mode="collect-pairs" if args.collect else "count-only",
                            backend=args.backend)
    rep = _run(a, b, cfg, args.epsilon)
    if args.format == "csv":
        print(CSV_HEADER)
        print(_csv_row(layout, axis, args.threads, 0, rep))
    else:
        print("backend=cuda")
        print(f"layout={layout.kind} k={layout.k} axis={axis} threads={args.threads}")
        print(f"result_count={rep.result_count}")
        print(f"partition_s={rep.partition_time:.6f}")
        print(f"sort_s={rep.sort_time:.6f}")
        print(f"join_s={rep.join_time:.6f}")
        print(f"total_s={rep.total_time:.6f}")
    if args.collect and args.pairs_out:
        np.save(args.pairs_out, rep.pairs)
    return 0


def cmd_bench(args) -> int:
    a, b, sa, sb = _load_pair(args.left, args.right)
    if args.reps < 1:
        print("error: --reps must be >= 1", file=sys.stderr)
        return 1
    print(CSV_HEADER)
    counts = set()
    for kind in args.layout_list.split(","):
        if kind not in ("1d", "2d"):
            print(f"error: unknown layout {kind!r}", file=sys.stderr)
            return 1
        axes = args.axis_list.split(",") if args.axis_list else [
            "auto" if kind == "1d" else "adaptive"]
        for kv in args.k_list.split(","):
            layout = PartitionLayout(kind, _resolve_k(kv, kind, sa, sb, args.epsilon))
            for axis in axes:
                if axis == "auto" and kind != "1d":
                    print(f"warning: skipping axis=auto for layout={kind} (stripes only)",
                          file=sys.stderr)
                    continue
                for threads in (int(t) for t in args.threads_list.split(",")):
                    cfg = engine.JoinConfig(layout=layout, axis_policy=axis, threads=threads,
                                            backend=args.backend)
                    for r in range(args.reps):
                        rep = _run(a, b, cfg, args.epsilon)
                        counts.add(rep.result_count)
                        print(_csv_row(layout, axis, threads, r, rep))
    if len(counts) > 1:
        print(f"error: result_count varied across configurations: {sorted(counts)}",
              file=sys.stderr)
        return 1
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_1908_11740_b200",
                                     description="B200 PBSM spatial join (filter step).")
    sub = parser.add_subparsers(dest="command", required=True)

    def inputs(p):
        p.add_argument("--left", required=True, help="left input (CSV or SJB1 binary)")
        p.add_argument("--right", required=True, help="right input")
        p.add_argument("--epsilon", type=float, default=None,
                       help="epsilon-distance join on point inputs")
        p.add_argument("--backend", choices=("cuda",), default=None)

    pj = sub.add_parser("join", help="run one spatial join")
    inputs(pj)
    pj.add_argument("--layout", choices=("1d", "2d"), default="1d")
    pj.add_argument("--k", default="auto")
    pj.add_argument("--axis", choices=("x", "y", "adaptive", "auto"), default=None)
    pj.add_argument("--threads", type=int, default=1)
    pj.add_argument("--collect", action="store_true")
    pj.add_argument("--pairs-out", default=None, help="with --collect: save pairs as .npy")
    pj.add_argument("--format", choices=("text", "csv"), default="text")
    pj.set_defaults(func=cmd_join)

    pb_ = sub.add_parser("bench", help="run a grid of configurations, emit CSV")
    inputs(pb_)
    pb_.add_argument("--layout-list", default="1d")
    pb_.add_argument("--k-list", default="auto")
    pb_.add_argument("--axis-list", default=None)
    pb_.add_argument("--threads-list", default="1")
    pb_.add_argument("--reps", type=int, default=1)
    pb_.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (SweepJoinError, OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
