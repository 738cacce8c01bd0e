#!/bin/bash
# split-K (latency configs): full GPU suite, then BERT-base bs 1 latency with split-K on / off
# (profiling build, Q4_KSPLIT=0 disables it) and the per-kernel launch list of 12 layers.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${1:-split_k or small or layer or drift}" > gpurun_out/ks_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ks_tests.log
for ks in "" 0 2 3 4 6 8; do
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_KSPLIT=$ks timeout -s KILL 120 python scripts/probe_latency.py 12 1 > gpurun_out/ks_lat_$ks.json 2>&1
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_KSPLIT=$ks timeout -s KILL 120 python scripts/probe_latency_w8.py 12 1 > gpurun_out/ks_lat_w8_$ks.json 2>&1
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ks_launches.csv \
  python scripts/probe_latency.py 12 1 > gpurun_out/ks_ncu.log 2>&1
Q4_KSPLIT=0 Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ks_launches_off.csv \
  python scripts/probe_latency.py 12 1 > gpurun_out/ks_ncu_off.log 2>&1
echo done
