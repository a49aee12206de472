#!/bin/bash
# trace build phase timings: TRACE_CFGS="c3 c2_4k" (default c3)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in ${TRACE_CFGS:-c3}; do
  echo "=== $cfg"
  DS_LIB=paper_2408_07092_b200/libds_trace.so timeout 300 python scripts/trace_phases.py $cfg > gpurun_out/trace_$cfg.log 2>&1
  grep -vE "^iter" gpurun_out/trace_$cfg.log | head -45
done
