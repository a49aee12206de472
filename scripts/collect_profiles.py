"""Copy one round's GPU evidence from gpurun_out/ (scripts/gpu_round.sh) into
profiles/: the bench JSON lines, the ncu launch list, the ncu --set full raw
pages of decode_kernel (native and 4-bit label) and the per-launch DRAM
traffic the bench reports as roofline.traffic.

usage: python scripts/collect_profiles.py [ROUND_TAG]   (default r1)
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT, PROF = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"

benches = {"bench.log": "bench_c3", "bench_ref.log": "bench_reference_c3", "bench_int4.log": "bench_c3_int4",
           "bench_offload_c5.log": "bench_offload_c5", "bench_clustered.log": "bench_c3_clustered",
           "bench_identity.log": "bench_c3_identity_pages"}
for c in ("c2_4k", "c2_16k", "c2_32k", "c4", "c5"):
    benches[f"bench_{c}.log"] = f"bench_{c}"
    benches[f"bench_{c}_int4.log"] = f"bench_{c}_int4"
for src, dst in benches.items():
    p = os.path.join(OUT, src)
    if not os.path.exists(p):
        continue
    try:  # the JSON line (warnings may precede it)
        line = json.loads([ln for ln in open(p) if ln.startswith("{")][-1])
    except Exception:
        continue
    json.dump(line, open(os.path.join(PROF, f"{tag}_{dst}.json"), "w"), indent=1)
    print("wrote", f"{tag}_{dst}.json")

if os.path.exists(os.path.join(OUT, "launches.csv")):
    shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_ncu_launches_c3.csv"))
    print("wrote", f"{tag}_ncu_launches_c3.csv")

ALG = {"c3": 201326592, "c3_int4": 159383552, "c2_32k": 50331648, "c4": 402653184, "c5": 201326592}
reps = [(f"prof_round_decode{s_}_raw.csv", "c3" + s_) for s_ in ("", "_int4")] + \
       [(f"prof_r2_{n}_raw.csv", n) for n in ALG]
for rep, name in reps:
    p = os.path.join(OUT, rep)
    if not os.path.exists(p):
        continue
    shutil.copy(p, os.path.join(PROF, f"{tag}_ncu_full_decode_kernel_{name}.csv"))
    rows = list(csv.reader(open(p)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name_):
        i = hdr.index(name_)
        v = float(vals[i])
        u = units[i]
        return v * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0) if "bytes" in name_ else v
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    alg = ALG[name]
    doc = {"config": name.replace("_int4", ""), "label": "int4" if name.endswith("_int4") else "native",
           "kernel": [v for h, v in zip(hdr, vals) if h == "Kernel Name"][0],
           "source": f"ncu --set full --clock-control none, 1 launch (profiles/{tag}_ncu_full_decode_kernel_{name}.csv)",
           "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch_group": int(rd + wr),
           "algorithmic_bytes": alg, "dram_over_algorithmic": round((rd + wr) / alg, 4),
           "gpu_time_us": get("gpu__time_duration.sum")}
    for m in ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "lts__t_sector_hit_rate.pct"):
        if m in hdr:
            doc[m] = get(m)
    json.dump(doc, open(os.path.join(PROF, f"traffic_{name}.json"), "w"), indent=1)
    print("wrote", f"traffic_{name}.json", doc["dram_over_algorithmic"])
for f in ("san_initcheck.log", "pytest_gpu.log", "smoke.log"):
    p = os.path.join(OUT, f)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(PROF, f"{tag}_{f}"))
