#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/smallm.jsonl
for pdl in "" 1; do
  for args in "4096 1024 1024 3 4" "8192 1024 1024 3 4" "4096 4096 1024 2 4" "8192 4096 1024 2 4" "4096 1024 4096 3 4" "4096 3072 1024 1 4"; do
    echo "pdl_off=$pdl $args" >> gpurun_out/smallm.jsonl
    if [ -n "$pdl" ]; then export Q4_NO_PDL=1; else unset Q4_NO_PDL; fi
    Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/smallm.jsonl 2>&1
  done
done
echo done
