"""Summarise an ncu --csv gpu__time_duration launch list: mean µs per kernel."""
import collections
import csv
import sys

rows = list(csv.DictReader(line for line in open(sys.argv[1]) if line.startswith('"')))
d = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        d[name].append(float(r["Metric Value"]))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, v in d.items():
    v = v[skip:] or v
    print(f"{k:28s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us")
