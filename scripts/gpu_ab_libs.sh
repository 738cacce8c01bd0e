#!/bin/bash
# A/B of two library builds on the layer kernels (probe_gemm / probe_attn / bs-1 latency)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/ab_libs.jsonl
for lib in libq4.so ${OTHER:-libq4_old.so} libq4.so ${OTHER:-libq4_old.so}; do
  echo "== $lib" >> gpurun_out/ab_libs.jsonl
  export Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib
  for args in "32768 4096 1024 2 4" "32768 1024 1024 3 4" "32768 1024 4096 3 4" "32768 3072 1024 1 4"; do
    timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/ab_libs.jsonl 2>&1
  done
  timeout -s KILL 60 python scripts/probe_attn.py >> gpurun_out/ab_libs.jsonl 2>&1
done
echo done
