#!/bin/bash
# RESLN_Q4 (O-proj / FFN2 shapes) epilogue anatomy: the profiling lib with Q4_DEBUG_SKIP knobs
# (32 = skip the cross-CTA rendezvous, 8 = skip epilogue math, 4 = skip the MMA)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/resln_probe.jsonl
for shape in "32768 1024 1024" "32768 1024 4096"; do
  timeout -s KILL 60 python scripts/probe_gemm.py $shape 3 4 >> gpurun_out/resln_probe.jsonl 2>>gpurun_out/resln_probe.err
  for k in ${KNOBS:-0 32 8 40 4}; do
    Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_DEBUG_SKIP=$k timeout -s KILL 60 python scripts/probe_gemm.py $shape 3 4 >> gpurun_out/resln_probe.jsonl 2>>gpurun_out/resln_probe.err
  done
done
echo done
