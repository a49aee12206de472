#!/bin/bash
# f1 offload line (L=32 pinned-host layers, link peaks, CUPTI overlap) + the N=2 one-GPU code path.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
free -g > gpurun_out/host_mem.txt; nproc >> gpurun_out/host_mem.txt
timeout 1200 python bench.py --offload --config c5 --steps 5 --warmup 2 > gpurun_out/bench_offload.log 2>&1; echo "offload rc=$?" >> gpurun_out/bench_offload.log
DS_BENCH_ONE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-dense --no-cpu-baseline --layers 2 \
  > gpurun_out/bench_n2_onegpu.log 2>&1; echo "n2 rc=$?" >> gpurun_out/bench_n2_onegpu.log
tail -2 gpurun_out/bench_offload.log | cut -c1-1500; tail -3 gpurun_out/bench_n2_onegpu.log | cut -c1-1500
