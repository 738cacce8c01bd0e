#!/bin/bash
# quick GPU iteration: selected GPU tests (-k expr in $1) + FFN1/O-proj/FFN2 probes
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${1:-gelu or layer or full_size}" > gpurun_out/i_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/i_tests.log
rm -f gpurun_out/i_probe.jsonl
for args in "32768 4096 1024 2 4" "32768 1024 1024 3 4" "32768 1024 4096 3 4"; do
  timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/i_probe.jsonl 2>>gpurun_out/i_probe.err
done
if [ -n "$2" ]; then timeout -s KILL 600 python bench.py --no-extras --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; fi
echo done
