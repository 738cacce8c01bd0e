#!/bin/bash
# ncu source-level captures of the row-epilogue GEMMs in isolation (FFN1 GELU_Q4, O-proj / FFN2 RESLN_Q4)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for args in "32768 4096 1024 2 4" "32768 1024 1024 3 4" "32768 1024 4096 3 4"; do
  timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/c_probe.jsonl 2>>gpurun_out/c_probe.err
done
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:w4a4_tc -s 4 -c 1 \
  -o gpurun_out/c_ffn1 python scripts/probe_gemm.py 32768 4096 1024 2 4 > gpurun_out/c_ncu1.log 2>&1
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:w4a4_tc -s 4 -c 1 \
  -o gpurun_out/c_oproj python scripts/probe_gemm.py 32768 1024 1024 3 4 > gpurun_out/c_ncu2.log 2>&1
echo done
