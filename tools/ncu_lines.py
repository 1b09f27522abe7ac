#!/usr/bin/env python
"""Attribute ncu warp-stall samples / executed instructions to CUDA source lines.

usage: ncu_lines.py REPORT.ncu-rep KERNEL_REGEX LIB.so [TOP]

ncu's CSV source page here carries metrics only for SASS; this maps each
SASS offset to its -lineinfo source line via nvdisasm and sums per line.
"""
import csv
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

rep, kre, lib = sys.argv[1], sys.argv[2], str(Path(sys.argv[3]).resolve())
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kname = rows[0][1]
st = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[st]
cs, ci = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
sass = []
for r in rows[st + 1:]:
    if not r or r[0] == "Address" or r[0] == "Kernel Name":
        break
    sass.append((int(r[0], 16), float(r[cs] or 0), float(r[ci] or 0)))
base = sass[0][0]

# mangled name of the profiled kernel → nvdisasm with line info
tmp = Path(tempfile.mkdtemp())
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cubins = list(tmp.glob("*.cubin"))
dis = subprocess.run(["nvdisasm", "-g", "-c", str(cubins[0])], capture_output=True, text=True).stdout
targs = re.findall(r"\((bool|int)\)(\d+)", kname)
want = ("I" + "".join(f"L{'b' if t == 'bool' else 'i'}{v}E" for t, v in targs) + "E") if targs else ""
short = kname.split("(")[0].split("::")[-1].split("<")[0]
line_of = {}
cur_fn = None
cur = None
for ln in dis.splitlines():
    mf = re.match(r"\s*\.text\.(\S+):", ln)
    if mf:
        cur_fn = mf.group(1)
        cur = None
        continue
    # mangled: <len><name>[template args]: "6k_join" does not match k_join_nested
    if cur_fn is None or f"{len(short)}{short}{want}" not in cur_fn:
        continue
    mm = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if mm:
        cur = (Path(mm.group(1)).name, int(mm.group(2)))
        continue
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if mo and cur is not None:
        line_of.setdefault(int(mo.group(1), 16), cur)
agg = defaultdict(lambda: [0.0, 0.0])
ts = ti = 0.0
for addr, s, i in sass:
    L = line_of.get(addr - base, -1)
    agg[L][0] += s
    agg[L][1] += i
    ts += s
    ti += i
csrc = Path(sys.argv[5] if len(sys.argv) > 5 else "/root/repo/paper_1908_11740_b200/csrc")
texts = {}
print(kname, f"samples={ts:.0f} inst={ti:.3e}")
for L, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    if L == -1:
        print(f"{'?':>20} stall {s / ts:6.3f} inst {i / ti:6.3f}")
        continue
    fname, line = L
    if fname not in texts:
        f = csrc / fname
        texts[fname] = f.read_text().splitlines() if f.exists() else []
    src = texts[fname]
    text = src[line - 1].strip()[:70] if 0 < line <= len(src) else "?"
    print(f"{fname + ':' + str(line):>20} stall {s / ts:6.3f} inst {i / ti:6.3f}  {text}")
