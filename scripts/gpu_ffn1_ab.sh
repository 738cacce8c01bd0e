#!/bin/bash
# FFN1 (GELU_Q4) epilogue A/B: product lib, then the profiling lib with Q4_DEBUG_SKIP knobs
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gelu" > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_tests.log
rm -f gpurun_out/ab_probe.jsonl
timeout -s KILL 60 python scripts/probe_gemm.py 32768 4096 1024 2 4 >> gpurun_out/ab_probe.jsonl 2>>gpurun_out/ab_probe.err
for k in ${KNOBS:-0 256 512 1024 768 1792 4}; do
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_DEBUG_SKIP=$k timeout -s KILL 60 python scripts/probe_gemm.py 32768 4096 1024 2 4 >> gpurun_out/ab_probe.jsonl 2>>gpurun_out/ab_probe.err
done
echo done
