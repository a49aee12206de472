#!/bin/bash
# A/B timing of experiment libraries: for each LIBS entry (paper_2408_07092_b200/<name>.so) and each
# SPECS entry "tag:bench args" (default c3), one bench line (decode-only roofline + step), twice.
# Logs -> gpurun_out/ab_<lib>_<tag>_<rep>.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
SPECS=${SPECS:-"c3:"}
for rep in 1 2; do
for spec in $SPECS; do
  tag=${spec%%:*}; args=${spec#*:}; args=${args//,/ }
  for L in ${LIBS:-libds}; do
    DS_LIB=paper_2408_07092_b200/$L.so timeout 300 python bench.py $args --no-cpu-baseline --no-e2e --no-dense-refs \
      --steps ${STEPS:-20} --warmup 5 > gpurun_out/ab_${L}_${tag}_$rep.log 2>&1
  done
done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f"{f:50s} us/launch {r.get('us_per_launch'):8.3f} frac {r.get('frac'):.4f} step_ms {d['ms_per_step']:.4f}")
PY
