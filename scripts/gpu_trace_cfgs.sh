#!/bin/bash
# Phase traces (libds_trace.so) of decode_kernel on several configs. Logs -> gpurun_out/trace_<cfg>.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for c in ${CFGS:-c2_32k c2_16k c4 c5}; do
  DS_LIB=paper_2408_07092_b200/libds_trace.so timeout 300 python scripts/trace_phases.py $c > gpurun_out/trace_$c.log 2>&1
done
for c in ${CFGS:-c2_32k c2_16k c4 c5}; do echo "== $c"; grep "dur \|sub \|iter 3" gpurun_out/trace_$c.log | head -40; done
