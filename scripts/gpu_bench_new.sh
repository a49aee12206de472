#!/bin/bash
# bench.py checks after a change: default c3 line (dense refs, pipelined e2e), the N=2 code path
# on one GPU (gloo, DS_BENCH_ONE_GPU=1), and the c2/c4 lines. Logs -> gpurun_out/
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python -c "import oracle; oracle.build()" > gpurun_out/oracle_build.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
DS_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-dense --no-cpu-baseline --layers 2 \
  > gpurun_out/bench_n2_onegpu.log 2>&1; echo "n2 rc=$?" >> gpurun_out/bench_n2_onegpu.log
for c in ${CFGS:-}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_$c.log 2>&1
done
tail -2 gpurun_out/bench.log | cut -c1-600; tail -4 gpurun_out/bench_n2_onegpu.log | cut -c1-600
