#!/bin/bash
# default bench line (with extras, cpu_baseline subprocess, strong-scaling model) + R4 parity
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "r4 or full_size or gelu or resln" > gpurun_out/bf_tests.log 2>&1
echo "rc=$?" >> gpurun_out/bf_tests.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bf_bench.json 2> gpurun_out/bf_bench.err
echo "bench rc=$?" >> gpurun_out/bf_tests.log
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bf_ref.json 2> gpurun_out/bf_ref.err
echo done
