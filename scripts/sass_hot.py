"""Aggregate an ncu SASS source page (--page source --csv --print-source sass):
runs of instructions with equal execution counts (basic blocks), ranked by
total warp instructions, with stall samples.  usage: sass_hot.py CSV [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
k = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
h = rows[k]
data = rows[k + 1:]
ie = h.index("Instructions Executed")
sm = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
tot = sum(int(r[ie] or 0) for r in data)
stot = sum(int(r[sm] or 0) for r in data)
print("total warp inst", tot, "stall samples", stot, "instructions", len(data))
runs, cur = [], None
for i, r in enumerate(data):
    c = int(r[ie] or 0)
    if cur and cur[1] == c:
        cur[2] += 1
        cur[3] += int(r[sm] or 0)
    else:
        cur = [i, c, 1, int(r[sm] or 0)]
        runs.append(cur)
runs.sort(key=lambda x: -(x[1] * x[2]))
for s, c, n, smp in runs[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"idx {s:5d} n={n:4d} exec={c:8d} total={c * n:10d} ({100 * c * n / tot:5.1f}%) samples={smp:6d} "
          f"({100 * smp / max(stot, 1):4.1f}%)  {data[s][src].strip()[:50]}")

if len(sys.argv) > 3:  # region stall breakdown: sass_hot.py CSV N a:b,c:d,...
    cols = [i for i, n in enumerate(h) if n.startswith("stall_")]
    for reg in sys.argv[3].split(","):
        a, b = map(int, reg.split(":"))
        tot_s = {h[i]: sum(int(r[i] or 0) for r in data[a:b]) for i in cols}
        ssum = sum(int(r[sm] or 0) for r in data[a:b])
        top = sorted(tot_s.items(), key=lambda x: -x[1])[:6]
        print(f"[{a}:{b}] samples {ssum} ({100 * ssum / max(stot, 1):.1f}%):", ", ".join(f"{k[6:]}={v}" for k, v in top))
