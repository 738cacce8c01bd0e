#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gelu or resln or layer or stack or split_k or bit_exact or linear or cluster or asym or w8a8" > gpurun_out/un_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/un_tests.log
rm -f gpurun_out/un.txt
for rep in 1 2 3; do echo "$(timeout -s KILL 120 python scripts/probe_latency.py 12 1 2>&1 | tail -1)" >> gpurun_out/un.txt; done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/un_bs1_launches.csv python scripts/probe_latency.py 12 1 > gpurun_out/un_ncu.log 2>&1
echo done
