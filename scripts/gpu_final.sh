#!/bin/bash
# full GPU suite + bench line + smoke (the round-end tiers, in this order)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/f_tests.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo "bench rc=$?" >> gpurun_out/f_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/f_tests.log
echo done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/f_bs1_launches.csv python scripts/probe_latency.py 12 1 > gpurun_out/f_ncu.log 2>&1
echo done2
