#!/bin/bash
# Profiling only: time each BERT-large layer GEMM with parts of the pipeline skipped
# (Q4_DEBUG_SKIP bits: 1 TMA, 2 unpack, 4 MMA, 8 epilogue math) to see which part bounds it.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for cfg in "32768 3072 1024 1" "32768 1024 1024 3" "32768 4096 1024 2" "32768 1024 4096 3"; do
  for sk in 0 8 2 10 4 12; do
    Q4_DEBUG_SKIP=$sk python scripts/probe_gemm.py $cfg 4
  done
done
