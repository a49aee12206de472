#!/bin/bash
# One iteration after a kernel change: GPU tests (PYTEST_ARGS), c3 phase trace, short c3 bench line
# (BENCH_ARGS), optional extra configs (CFGS). Logs -> gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > gpurun_out/oracle_build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for c in ${TRACE_CFGS:-c3}; do
  DS_LIB=paper_2408_07092_b200/libds_trace.so timeout 300 python scripts/trace_phases.py $c > gpurun_out/trace_$c.log 2>&1
  echo "== trace $c"; grep "dur \|sub \|iter 3" gpurun_out/trace_$c.log | head -40
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-dense-refs ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ${CFGS:-}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 --no-e2e --no-dense-refs > gpurun_out/bench_$c.log 2>&1
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/bench*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line); r = d["roofline"]
            print(f, d["config"]["workload"], "us/launch", r.get("us_per_launch"), "frac", r.get("frac"), "step ms", d["ms_per_step"], "value", d["value"])
PY
