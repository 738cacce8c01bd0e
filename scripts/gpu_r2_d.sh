#!/bin/bash
# full GPU suite + bench line; bs-1 GEMM epilogue phase traces; R4 / TN A-B for the O-proj shape
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/d_tests.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
echo "bench rc=$?" >> gpurun_out/d_tests.log
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/d_trace.bin gpurun_out/d_probe.jsonl
for args in "128 768 768 3 4" "128 768 3072 3 4" "128 3072 768 2 4" "128 2304 768 1 4"; do
  Q4_LIB_PATH=$P Q4_TRACE=gpurun_out/d_trace.bin timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/d_probe.jsonl 2>&1
done
python scripts/trace_report.py gpurun_out/d_trace.bin > gpurun_out/d_trace.txt 2>&1; rm -f gpurun_out/d_trace.bin
for args in "32768 1024 1024 3 4" "32768 1024 4096 3 4" "32768 4096 1024 2 4"; do
  Q4_LIB_PATH=$P timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/d_probe.jsonl 2>&1
  Q4_LIB_PATH=$P Q4_R4=1 timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/d_probe.jsonl 2>&1
done
echo done
