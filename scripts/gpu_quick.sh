#!/bin/bash
# quick iteration: gpu tests + trace + bench (short) + launch list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
if [[ -f paper_2408_07092_b200/libds_trace.so ]]; then
  DS_LIB=paper_2408_07092_b200/libds_trace.so timeout 300 python scripts/trace_phases.py ${TRACE_CFG:-c3} > gpurun_out/trace.log 2>&1
  grep -vE "^iter" gpurun_out/trace.log | grep -E "dur|span|Error|error" | head -30
fi
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.log").read().splitlines()[0])
    print({k: d.get(k) for k in ["value", "us_per_layer", "dense_us_per_layer", "speedup_vs_dense"]}, d["roofline"]["frac"], d.get("clocks"))
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.log").read()[-2000:])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:ds:: -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 2 --no-dense --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/launches.py gpurun_out/launches.csv | grep -v calibrate
