#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
rm -f gpurun_out/f2_trace.bin gpurun_out/f2_trace.txt
for args in "128 768 3072 3 4" "128 768 768 3 4"; do
  PROBE_GRAPH= Q4_LIB_PATH=$P Q4_TRACE=gpurun_out/f2_trace.bin timeout -s KILL 60 python scripts/probe_gemm.py $args > /dev/null 2>&1
  python scripts/trace_report.py gpurun_out/f2_trace.bin | sort | uniq -c | sort -rn | head -3 >> gpurun_out/f2_trace.txt
  echo "-- $args" >> gpurun_out/f2_trace.txt
  rm -f gpurun_out/f2_trace.bin
done
echo done
