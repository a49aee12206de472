#!/bin/bash
# Full ncu capture of the decode kernels (one launch each) for one bench config.
# usage: ncu_full.sh OUTNAME [KERNEL_REGEX] [-- extra bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=${1:-prof}; shift
KREGEX="score_select|attn_kernel|ds_fused"
if [[ $# -gt 0 && $1 != "--" ]]; then KREGEX=$1; shift; fi
[[ ${1:-} == "--" ]] && shift
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:$KREGEX" -c ${NCU_COUNT:-3} -o gpurun_out/$OUT -f \
  python bench.py --steps 1 --warmup 1 --layers 1 --no-dense --no-e2e --no-cpu-baseline "$@" > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$OUT.log
tail -3 gpurun_out/$OUT.log
