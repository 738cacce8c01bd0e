#!/bin/bash
# full GPU test suite + default bench line (with extras) + reference arm
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rd_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rd_tests.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/rd_bench.json 2> gpurun_out/rd_bench.err
echo "bench rc=$?" >> gpurun_out/rd_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rd_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/rd_tests.log
echo done
