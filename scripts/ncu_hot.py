"""Summarise an ncu source page (SASS) export: top instructions by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((int(r[wi]), i, r[si].strip()))
    except Exception:
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, i, src in sorted(data, reverse=True)[:n]:
    print(f"{s:6d} {100*s/tot:5.1f}%  [{i:4d}] {src[:100]}")
