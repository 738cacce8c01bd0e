#!/bin/bash
# Profiling only: A/B the per-kernel bench breakdown between paper_2301_12017_b200/libq4_old.so
# and the in-tree build (two alternating rounds each).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do
for lib in libq4_old.so libq4.so; do
  echo "== $lib"
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib bash scripts/quick_bench.sh
done
done
