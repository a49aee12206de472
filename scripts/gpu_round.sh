#!/bin/bash
# Round evidence: full GPU tests + smoke, default bench (with cpu_baseline), extra configs,
# ncu launch list and one ncu --set full capture of decode_kernel (c3).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > gpurun_out/oracle_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in c2_4k c2_16k c2_32k c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 --no-e2e --layers 4 > gpurun_out/bench_$c.log 2>&1
done
# f2: the 4-bit label on the same configs
timeout 600 python bench.py --label int4 --no-cpu-baseline > gpurun_out/bench_int4.log 2>&1
for c in c2_32k c4 c5; do
  timeout 300 python bench.py --config $c --label int4 --no-cpu-baseline --steps 10 --warmup 3 --no-e2e --layers 4 > gpurun_out/bench_${c}_int4.log 2>&1
done
timeout 600 python bench.py --offload --config c5 --no-cpu-baseline > gpurun_out/bench_offload_c5.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:ds:: -c 200 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 2 --no-dense --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
NCU_COUNT=1 timeout 900 bash scripts/ncu_full.sh prof_round_decode decode_kernel
NCU_COUNT=1 timeout 900 bash scripts/ncu_full.sh prof_round_decode_int4 decode_kernel -- --label int4
for f in prof_round_decode prof_round_decode_int4; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null
done
for f in gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/ncu_launch.log; do echo "== $f"; tail -n 2 $f | cut -c1-400; done
