#!/bin/bash
# Profiling only: A/B the FFN1 GEMM (M=32768, N=4096, K=1024, GELU_Q4, W8) and the bench step
# between the in-tree build and paper_2301_12017_b200/libq4_old.so.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for lib in libq4_old.so libq4.so; do
  echo "== $lib"
  export Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib
  python scripts/probe_gemm.py 32768 4096 1024 2 4
  bash scripts/quick_bench.sh | grep -E "seq/s|ffn1"
done
