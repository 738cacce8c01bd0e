#!/bin/bash
# row-epilogue rendezvous A/B: row-epilogue parity tests, large-M row GEMMs, bs-1 latency, traces
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${1:-gelu or resln or layer or split_k or full_size or r4 or nccl or asym or w8a8 or pipeline or stack}" > gpurun_out/x_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/x_tests.log
rm -f gpurun_out/x_probe.jsonl gpurun_out/x_trace.bin
for args in "32768 1024 1024 3 4" "32768 1024 4096 3 4" "32768 4096 1024 2 4"; do
  for i in 1 2; do timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/x_probe.jsonl 2>&1; done
done
for i in 1 2 3; do timeout -s KILL 120 python scripts/probe_latency.py 12 1 >> gpurun_out/x_lat.json 2>&1; done
P=$PWD/paper_2301_12017_b200/libq4_prof.so
for args in "128 768 768 3 4" "128 768 3072 3 4" "128 3072 768 2 4" "32768 4096 1024 2 4" "32768 1024 1024 3 4"; do
  Q4_LIB_PATH=$P Q4_TRACE=gpurun_out/x_trace.bin timeout -s KILL 60 python scripts/probe_gemm.py $args > /dev/null 2>&1
done
python scripts/trace_report.py gpurun_out/x_trace.bin > gpurun_out/x_trace.txt 2>&1; rm -f gpurun_out/x_trace.bin
echo done
