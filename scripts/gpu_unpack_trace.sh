#!/bin/bash
# unpack-warp anatomy at M = 128 (trace slot 63: per k-block wait_full_p / wait_empty_u / unpack /
# fence+arrive, averaged over k-blocks 16..), split-K off so one CTA runs the whole k-loop
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/u_trace.bin
for args in "128 768 4096 3 4" "128 768 4096 1 4" "32768 1024 4096 3 4"; do
  Q4_KSPLIT=0 Q4_LIB_PATH=$P Q4_TRACE=gpurun_out/u_trace.bin PROBE_GRAPH= timeout -s KILL 60 python scripts/probe_gemm.py $args > /dev/null 2>&1
  python scripts/trace_report.py gpurun_out/u_trace.bin | grep -i "unpack\|mma" | sort | uniq -c | head -6 >> gpurun_out/u_trace.txt
  echo "-- $args" >> gpurun_out/u_trace.txt
  rm -f gpurun_out/u_trace.bin
done
echo done
