#!/bin/bash
# attention A/B: libq4.so (this tree) vs libq4_ab.so (saved build) -- probe at B = 256, bench step
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or layer or stack" > gpurun_out/aa_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/aa_tests.log
rm -f gpurun_out/aa.txt
for rep in 1 2 3; do
  for lib in libq4.so libq4_ab.so; do
    echo "$lib $(Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib timeout -s KILL 60 python scripts/probe_attn.py 2>&1 | tail -1)" >> gpurun_out/aa.txt
  done
done
for lib in libq4.so libq4_ab.so; do
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/aa_bench_$lib.json 2>/dev/null
  echo "$lib $(python -c "import json; d=json.load(open('gpurun_out/aa_bench_$lib.json')); print(round(d['value']), {k: round(v['ms']*1e3,1) for k, v in d['kernels'].items()})")" >> gpurun_out/aa.txt
  echo "$lib $(Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib timeout -s KILL 120 python scripts/probe_latency.py 12 1 2>&1 | tail -1)" >> gpurun_out/aa.txt
done
echo done
