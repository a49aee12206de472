"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, gi, bi = (hdr.index(x) for x in ("Kernel Name", "Metric Value", "Grid Size", "Block Size"))
agg = collections.OrderedDict()
for r in rows:
    key = (r[ki].split("(")[0].replace("void ", "")[:70], r[gi], r[bi])
    agg.setdefault(key, []).append(float(r[vi]) / 1000.0)
for (name, grid, block), v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v):9.2f} us  {name} grid={grid} block={block}")
