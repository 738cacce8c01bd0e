#!/bin/bash
# ncu launch lists of the 12-layer BERT-base bs-1 forward: W4A4 vs W8A8 (per-kernel latency)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat4.csv \
  python scripts/probe_latency.py 12 1 > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat8.csv \
  python scripts/probe_latency_w8.py 12 > /dev/null 2>&1
echo done
