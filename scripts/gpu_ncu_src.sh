#!/bin/bash
# One ncu --set full capture (source counters) of decode_kernel on a bench config,
# exported as the raw page and the SASS source page. usage: gpu_ncu_src.sh NAME [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NAME=${1:-src_c3}; shift
NCU_COUNT=1 timeout 900 bash scripts/ncu_full.sh $NAME decode_kernel -- "$@"
ncu -i gpurun_out/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>/dev/null
ncu -i gpurun_out/$NAME.ncu-rep --page source --csv --print-source sass > gpurun_out/${NAME}_sass.csv 2>/dev/null
ls -la gpurun_out/$NAME*
