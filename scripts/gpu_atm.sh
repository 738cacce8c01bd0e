#!/bin/bash
# A-in-TMEM narrow-tile mainloop: small-M parity, latency A/B against libq4_ab.so, launch list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 700 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${1:-bit_exact or extreme or linear or split_k or layer or stack or pipeline or quantize}" > gpurun_out/t_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/t_tests.log
rm -f gpurun_out/t_lat.txt
for rep in 1 2; do
  for lib in libq4.so libq4_ab.so; do
    echo "$lib $(Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib timeout -s KILL 120 python scripts/probe_latency.py 12 1 2>&1 | tail -1) $(Q4_LIB_PATH=$PWD/paper_2301_12017_b200/$lib timeout -s KILL 120 python scripts/probe_latency_w8.py 12 2>&1 | tail -1)" >> gpurun_out/t_lat.txt
  done
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/t_bs1_launches.csv python scripts/probe_latency.py 12 1 > gpurun_out/t_ncu.log 2>&1
echo done
