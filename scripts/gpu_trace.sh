cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
DS_LIB=paper_2408_07092_b200/libds_trace.so timeout 300 python scripts/trace_phases.py c3 > gpurun_out/trace.log 2>&1
grep -vE "^iter" gpurun_out/trace.log | head -40
