#!/bin/bash
# Round-2 evidence on one B200: GPU tests + smoke, bench lines for every config (16-bit and 4-bit
# label, iid / clustered, random / identity pages), offload, reference arm, ncu launch list of the
# default bench, ncu --set full of decode_kernel on c3 / c3 int4 / c2_32k / c4 / c5, and
# compute-sanitizer initcheck. Logs -> gpurun_out/ (collected by scripts/collect_profiles.py r2).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
STAGE=${1:-all}
python -c "import oracle; oracle.build()" > gpurun_out/oracle_build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $STAGE == all || $STAGE == test ]]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [[ $STAGE == all || $STAGE == bench ]]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
  timeout 600 python bench.py --label int4 --no-cpu-baseline > gpurun_out/bench_int4.log 2>&1
  timeout 600 python bench.py --structure clustered --no-cpu-baseline --no-e2e --no-dense-refs > gpurun_out/bench_clustered.log 2>&1
  timeout 600 python bench.py --pages identity --no-cpu-baseline --no-e2e --no-dense-refs > gpurun_out/bench_identity.log 2>&1
  for c in c2_4k c2_16k c2_32k c4 c5; do
    timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_$c.log 2>&1
  done
  for c in c2_32k c4 c5; do
    timeout 600 python bench.py --config $c --label int4 --no-cpu-baseline --steps 10 --warmup 3 --no-e2e --no-dense-refs > gpurun_out/bench_${c}_int4.log 2>&1
  done
  timeout 1200 python bench.py --offload --config c5 --steps 5 --warmup 2 > gpurun_out/bench_offload_c5.log 2>&1
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
fi
if [[ $STAGE == all || $STAGE == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:ds:: -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-dense --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
  for spec in "c3:" "c3_int4:--label int4" "c2_32k:--config c2_32k" "c4:--config c4" "c5:--config c5"; do
    name=${spec%%:*}; args=${spec#*:}
    NCU_COUNT=1 timeout 900 bash scripts/ncu_full.sh prof_r2_$name decode_kernel -- --no-dense-refs $args > /dev/null 2>&1
    ncu -i gpurun_out/prof_r2_$name.ncu-rep --page raw --csv > gpurun_out/prof_r2_${name}_raw.csv 2>/dev/null
    mv gpurun_out/prof_r2_$name.ncu-rep /tmp/ 2>/dev/null  # (reports stay on the box: gpurun_out <= 64 MiB)
  done
fi
if [[ $STAGE == all || $STAGE == san ]]; then
  timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/san_initcheck.log 2>&1
  echo "initcheck rc=$?" >> gpurun_out/san_initcheck.log
fi
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/ncu_launch.log gpurun_out/san_initcheck.log; do
  [[ -f $f ]] && { echo "== $f"; tail -n 2 $f | cut -c1-300; }
done
