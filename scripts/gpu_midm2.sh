#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/midm2.jsonl
for M in 2048 4096 6144 8192; do
  for tn in 256 128; do
    for pdl in "" 1; do
      echo "TN=$tn NOPDL=$pdl" >> gpurun_out/midm2.jsonl
      if [ -n "$pdl" ]; then export Q4_NO_PDL=1; else unset Q4_NO_PDL; fi
      for rep in 1 2; do
        Q4_LIB_PATH=$P Q4_TN=$tn timeout -s KILL 60 python scripts/probe_gemm.py $M 1024 1024 3 4 >> gpurun_out/midm2.jsonl 2>&1
      done
    done
  done
done
unset Q4_NO_PDL
for M in 4096 8192; do
  for tn in 256 128; do
    echo "GELU TN=$tn" >> gpurun_out/midm2.jsonl
    Q4_LIB_PATH=$P Q4_TN=$tn timeout -s KILL 60 python scripts/probe_gemm.py $M 4096 1024 2 4 >> gpurun_out/midm2.jsonl 2>&1
  done
done
echo done
