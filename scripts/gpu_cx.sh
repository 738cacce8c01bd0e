#!/bin/bash
# CX (single-m-block row GEMMs as one cluster, DSMEM exchange): parity, latency A/B, launch list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gelu or resln or layer or stack or asym or w8a8 or split_k or pipeline or degenerate or clip" > gpurun_out/cx_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/cx_tests.log
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/cx.txt
for rep in 1 2; do
  for cx in 1 0; do
    echo "CX=$cx $(Q4_LIB_PATH=$P Q4_CX=$cx timeout -s KILL 120 python scripts/probe_latency.py 12 1 2>&1 | tail -1) $(Q4_LIB_PATH=$P Q4_CX=$cx timeout -s KILL 120 python scripts/probe_latency_w8.py 12 2>&1 | tail -1)" >> gpurun_out/cx.txt
  done
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/cx_bs1_launches.csv python scripts/probe_latency.py 12 1 > gpurun_out/cx_ncu.log 2>&1
echo done
