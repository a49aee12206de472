cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.log
timeout 900 python -m pytest tests -q -m gpu --timeout 300 --durations=12 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
DS_LIB=paper_2408_07092_b200/libds_trace.so timeout 300 python scripts/trace_phases.py c3 > gpurun_out/trace_c3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log | cut -c1-3000
