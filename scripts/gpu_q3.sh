#!/bin/bash
# Q3 row kernels (TN = 128, three accumulators, A in TMEM) at large M: parity with the knob on
# (profiling build), GEMM A/B with graph replay, bench step A/B
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
P=$PWD/paper_2301_12017_b200/libq4_prof.so
Q4_LIB_PATH=$P Q4_Q3=1 timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  -k "gelu or resln or full_size or layer or stack or r4 or asym" > gpurun_out/q3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/q3_tests.log
rm -f gpurun_out/q3_probe.txt
for args in "32768 1024 1024 3" "32768 1024 4096 3" "32768 4096 1024 2" "8192 1024 1024 3" "8192 1024 4096 3" "8192 4096 1024 2"; do
  for q3 in 0 1; do
    echo "Q3=$q3 $(PROBE_GRAPH=1 Q4_LIB_PATH=$P Q4_Q3=$q3 timeout -s KILL 60 python scripts/probe_gemm.py $args 4 2>&1 | tail -1)" >> gpurun_out/q3_probe.txt
  done
done
for q3 in 0 1; do
  Q4_LIB_PATH=$P Q4_Q3=$q3 timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/q3_bench_$q3.json 2>/dev/null
  echo "Q3=$q3 $(python -c "import json; d=json.load(open('gpurun_out/q3_bench_$q3.json')); print(round(d['value']), {k: round(v['ms']*1e3,1) for k, v in d['kernels'].items()})")" >> gpurun_out/q3_probe.txt
done
echo done
