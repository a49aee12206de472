#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list. Logs -> gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import oracle; oracle.build()" > gpurun_out/oracle_build.log 2>&1
STAGE=${1:-all}
if [[ $STAGE == all || $STAGE == test ]]; then
  timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [[ $STAGE == all || $STAGE == bench ]]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
if [[ $STAGE == all || $STAGE == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:ds:: -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 2 --no-dense --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
fi
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 $f; done
