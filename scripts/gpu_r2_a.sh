#!/bin/bash
# round-2 baseline: bench (no extras), INT8 ceiling, ncu source captures of FFN1 / O-proj in isolation
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout -s KILL 300 python bench.py --no-extras --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
timeout -s KILL 120 python scripts/int8_ceiling.py gpurun_out/a_int8.json > /dev/null 2> gpurun_out/a_int8.err
for args in "32768 4096 1024 2 4" "32768 1024 1024 3 4" "32768 1024 4096 3 4"; do
  timeout -s KILL 60 python scripts/probe_gemm.py $args >> gpurun_out/a_probe.jsonl 2>>gpurun_out/a_probe.err
done
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:w4a4_tc -s 4 -c 1 \
  -o gpurun_out/a_ffn1 python scripts/probe_gemm.py 32768 4096 1024 2 4 > gpurun_out/a_ncu1.log 2>&1
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:w4a4_tc -s 4 -c 1 \
  -o gpurun_out/a_oproj python scripts/probe_gemm.py 32768 1024 1024 3 4 > gpurun_out/a_ncu2.log 2>&1
echo done
