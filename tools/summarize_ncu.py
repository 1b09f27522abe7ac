#!/usr/bin/env python
"""Summarise an ncu launch list (CSV) and/or a --set full report into markdown.

usage: summarize_ncu.py --launches launches.csv [--full prof.ncu-rep] [--title T] > out.md
"""
import argparse
import collections
import csv
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("--launches")
ap.add_argument("--full")
ap.add_argument("--title", default="ncu summary")
a = ap.parse_args()
print(f"# {a.title}\n")
if a.launches:
    rows = list(csv.reader(open(a.launches)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        agg[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print("## Launch list (gpu__time_duration.sum, cold-cache, serialised)\n")
    print("| kernel | launches | mean µs | share |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    print()
if a.full:
    out = subprocess.run(["ncu", "-i", a.full, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    keys = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
            ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
    print("## Full-set captures\n")
    print("| kernel | " + " | ".join(k[1] for k in keys) + " | top stalls |")
    print("|---" * (len(keys) + 2) + "|")
    units = rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
        vals = []
        for k, _ in keys:
            i = h.index(k)
            vals.append(f"{r[i]} {units[i]}".strip())
        st = [(float(r[i]), n) for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled")
              and n.endswith("per_issue_active.ratio") and r[i] not in ("", "n/a")]
        st.sort(reverse=True)
        top = ", ".join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.1f}"
                        for v, n in st[:3])
        print(f"| `{name}` | " + " | ".join(vals) + f" | {top} |")
