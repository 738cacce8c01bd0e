#!/bin/bash
# Round profile evidence (run under gpurun; outputs in gpurun_out/, summarised into profiles/):
#  1. ncu launch list (gpu__time_duration, clocks not locked) of the bench command
#  2. one `ncu --set full` capture of the dominant kernel (FFN1 GELU_Q4 GEMM, W8 variant)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${1:-r2}
B="python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
  --log-file gpurun_out/${R}_launches.csv $B > gpurun_out/${R}_ncu_list.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k regex:"ILi256ELi2ELb1ELb0" -s 1 -c 1 -o gpurun_out/${R}_ffn1 \
  python bench.py --steps 2 --warmup 1 --layers 1 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/${R}_ncu_full.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k regex:"attention|w4a4" -s 0 -c 5 -o gpurun_out/${R}_layer \
  python bench.py --steps 2 --warmup 1 --layers 1 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/${R}_ncu_layer.log 2>&1
echo done
