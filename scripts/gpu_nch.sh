#!/bin/bash
# Cluster-size sweep (libds_nch.so: built with -DDS_EXP_NCH_ENV, DS_NCH forces the CTAs per unit).
# SPECS entries "config:n1,n2,..."; one decode-only bench line per (config, nch). Logs -> gpurun_out/nch_*.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for spec in ${SPECS:-c2_4k:1,2,4 c2_16k:1,2,4 c2_32k:2,4 c4:1,2}; do
  c=${spec%%:*}; ns=${spec#*:}
  for n in ${ns//,/ }; do
    DS_NCH=$n DS_LIB=paper_2408_07092_b200/libds_nch.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e \
      --no-dense-refs --steps 10 --warmup 3 > gpurun_out/nch_${c}_$n.log 2>&1
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/nch_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f"{f:40s} us/launch {r.get('us_per_launch'):8.3f} frac {r.get('frac'):.4f} step_ms {d['ms_per_step']:.4f}")
PY
