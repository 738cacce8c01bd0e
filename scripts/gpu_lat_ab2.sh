#!/bin/bash
# latency knobs after the A-in-TMEM change: split-K slices for FFN2, TN = 32 for the F16 QKV
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/ab2.txt
for rep in 1 2; do
  for cfg in "X=1" "Q4_KSPLIT=6" "Q4_KSPLIT=8" "Q4_KSPLIT=4" "Q4_TN=32"; do
    echo "$cfg $(env Q4_LIB_PATH=$P $cfg timeout -s KILL 120 python scripts/probe_latency.py 12 1 2>&1 | tail -1)" >> gpurun_out/ab2.txt
  done
done
echo done
