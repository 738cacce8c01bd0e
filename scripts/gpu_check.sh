#!/bin/bash
# Run the GPU test groups as separate processes (a kernel fault poisons its CUDA context),
# each under a hard timeout.  Logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu.txt 2>&1
for k in ${@:-quantize exhaustive gemm_i32 extreme linear_f16 gelu resln degenerate requant attention teacher stack full_size launch}; do
  echo "=== $k" >> gpurun_out/gpu_tests.log
  timeout -s KILL ${T:-600} python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$k" -x > gpurun_out/.group.log 2>&1
  rc=$?
  tail -25 gpurun_out/.group.log >> gpurun_out/gpu_tests.log
  echo "rc=$rc" >> gpurun_out/gpu_tests.log
done
