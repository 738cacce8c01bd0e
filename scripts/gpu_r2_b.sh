#!/bin/bash
# round-2 first GPU pass: full GPU test suite, default bench line, INT8 ceiling
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b_smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/b_tests.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
timeout -s KILL 120 python scripts/int8_ceiling.py gpurun_out/b_int8.json > /dev/null 2> gpurun_out/b_int8.err
echo done
