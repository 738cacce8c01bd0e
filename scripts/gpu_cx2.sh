#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/cx2.txt
for rep in 1 2; do
  for cfg in "X=1" "Q4_KSPLIT=0" "Q4_KSPLIT=4" "Q4_KSPLIT=2"; do
    echo "$cfg $(env Q4_LIB_PATH=$P $cfg timeout -s KILL 120 python scripts/probe_latency.py 12 1 2>&1 | tail -1)" >> gpurun_out/cx2.txt
  done
done
for cfg in "X=1" "Q4_KSPLIT=0"; do
  echo "FFN2 $cfg $(env PROBE_GRAPH=1 Q4_LIB_PATH=$P $cfg timeout -s KILL 60 python scripts/probe_gemm.py 128 768 3072 3 4 2>&1 | tail -1)" >> gpurun_out/cx2.txt
done
echo done
