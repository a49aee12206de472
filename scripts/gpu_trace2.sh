#!/bin/bash
# trace phases with a given trace library: TRACE_LIBS="a.so b.so" TRACE_CFGS="c3"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for lib in ${TRACE_LIBS:-paper_2408_07092_b200/libds_trace.so}; do
for cfg in ${TRACE_CFGS:-c3}; do
  echo "=== $lib $cfg"
  DS_LIB=$lib timeout 300 python scripts/trace_phases.py $cfg > gpurun_out/trace_$cfg.log 2>&1
  grep -A25 "fused decode" gpurun_out/trace_$cfg.log | grep -E "dur|sub"
done; done
