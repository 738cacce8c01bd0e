#!/bin/bash
# mid-size M (the per-rank sizes of the strong-scaling model): row / F16 GEMMs at TN = 256 vs 128
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/midm.jsonl
for M in 2048 4096 8192 16384; do
  for shape in "1024 1024 3" "4096 1024 2" "1024 4096 3" "3072 1024 1"; do
    for tn in 256 128; do
      echo "TN=$tn" >> gpurun_out/midm.jsonl
      PROBE_GRAPH=1 Q4_LIB_PATH=$P Q4_TN=$tn timeout -s KILL 60 python scripts/probe_gemm.py $M $shape 4 >> gpurun_out/midm.jsonl 2>&1
    done
  done
done
echo done
