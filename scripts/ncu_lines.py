"""Aggregate an ncu SASS source-page export by CUDA source line.

usage: python scripts/ncu_lines.py SASS_CSV CUBIN_DIS FUNCTION [N]
  SASS_CSV  : ncu -i rep --page source --csv --print-source sass
  CUBIN_DIS : nvdisasm -g -c <cubin> (line-annotated disassembly)
Prints the top source lines by warp-stall samples with their top stall reasons.
"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dis, fn = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40

lines = open(dis).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(fn + ":"))
off2src = {}
cur = None
for l in lines[start + 2:]:
    if re.match(r"^\S.*:$", l) and not l.startswith(".text"):
        if not l.startswith(".L"):
            break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2src[int(m.group(1), 16)] = cur

rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ai, si = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
base = int(rows[2][ai], 16)
agg = defaultdict(lambda: [0, 0, defaultdict(int)])
for r in rows[2:]:
    try:
        off = int(r[ai], 16) - base
        s = int(r[si])
    except (ValueError, IndexError):
        continue
    key = off2src.get(off, ("?", 0))
    a = agg[key]
    a[0] += s
    a[1] += int(r[ei] or 0)
    for i, h in stall_cols:
        try:
            a[2][h] += int(r[i])
        except ValueError:
            pass
tot = sum(a[0] for a in agg.values())
src = {}
for f in set(k[0] for k in agg):
    for path in ("paper_2408_07092_b200/csrc/" + f,):
        try:
            src[f] = open(path).read().splitlines()
        except OSError:
            pass
print(f"total stall samples {tot}")
for (f, ln), (s, ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    txt = src.get(f, [""] * (ln + 1))[ln - 1].strip() if f in src and ln > 0 else ""
    why = ", ".join(f"{h[6:]}={v}" for h, v in top if v)
    print(f"{s:6d} {100 * s / tot:5.1f}%  {f}:{ln:<5d} {txt[:70]:70s} | {why}")
