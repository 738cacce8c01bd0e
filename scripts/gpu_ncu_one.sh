#!/bin/bash
# one ncu --set full capture (source counters) of a probe_gemm launch: SHAPE="M N K kind mainloop", OUT=name
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 500 ncu --set full --clock-control none --import-source on -k regex:w4a4_tc -s 4 -c 1 \
  -o gpurun_out/${OUT:-n_one} python scripts/probe_gemm.py ${SHAPE:-32768 4096 1024 2 4} > gpurun_out/${OUT:-n_one}.log 2>&1
echo done
