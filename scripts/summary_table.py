"""Markdown rows of the measured table (README) from profiles/r2_bench_*.json."""
import json
import os

P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def load(name):
    p = os.path.join(P, f"r2_bench_{name}.json")
    return json.load(open(p)) if os.path.exists(p) else None


rows = [("**c3** (128 units, S=32K)", "c3", "c3_int4"), ("c3 clustered selection", "c3_clustered", None),
        ("c3 identity page order", "c3_identity_pages", None), ("c2 S=4K (32 MHA units, B=1)", "c2_4k", None),
        ("c2 S=16K", "c2_16k", None), ("c2 S=32K", "c2_32k", "c2_32k_int4"),
        ("c4 (512 units, S=16K)", "c4", "c4_int4"), ("c5 (32 units, S=128K)", "c5", "c5_int4")]
for label, n, n4 in rows:
    d = load(n)
    if not d:
        continue
    r = d["roofline"]
    d4 = load(n4) if n4 else None
    fd = d.get("speedup_vs_fastest_dense")
    q4 = f"{d4['roofline']['us_per_launch']:.1f} ({d4['roofline']['frac']:.3f})" if d4 else "—"
    print(f"| {label} | {r['us_per_launch']:.2f} | {r['frac']:.3f} | {d.get('speedup_vs_dense') or 0:.2f}× | "
          f"{(f'{fd:.2f}×' if fd else '—')} | {q4} |")
d = load("c3")
if d:
    r = d["roofline"]
    print("\nc3:", {k: r.get(k) for k in ("achieved", "peak", "frac", "us_per_launch", "cupti_us_per_launch", "cupti_frac",
                                         "isolated_us", "isolated_frac", "traffic")})
    print("step us/layer", d["us_per_layer"], "ms/step", d["ms_per_step"], "value", d["value"])
    print("e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "dense refs",
          {k: v.get("us_per_layer") for k, v in d.get("dense_refs", {}).items()})
    print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"].get("one_core", {}).get("value"))
