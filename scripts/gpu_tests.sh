#!/bin/bash
# GPU test run only: pytest -m gpu (optionally a -k filter via PYTEST_ARGS)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 240 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "passed|failed|Error|error|assert" gpurun_out/pytest_gpu.log | head -40
