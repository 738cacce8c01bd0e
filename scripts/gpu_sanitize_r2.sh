#!/bin/bash
# compute-sanitizer over the round-2 kernels: memcheck on the sparse / asymmetric / R4 parity tests,
# racecheck on the sparse GEMM and an asymmetric row-epilogue GEMM (small shapes)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/sanitizer_r2
CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_sparse.py -m gpu -q -x -p no:cacheprovider \
  -k "extreme or 100-768" > gpurun_out/sanitizer_r2/memcheck_sparse.log 2>&1
timeout -s KILL 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_asym.py -m gpu -q -x -p no:cacheprovider \
  -k "teacher_forced and base or attention_asym_codes and 3-77" > gpurun_out/sanitizer_r2/memcheck_asym.log 2>&1
timeout -s KILL 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_sparse.py -m gpu -q -x -p no:cacheprovider \
  -k "100-768" > gpurun_out/sanitizer_r2/racecheck_sparse.log 2>&1
timeout -s KILL 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_asym.py -m gpu -q -x -p no:cacheprovider \
  -k "symmetric_input_asymmetric_output and 37" > gpurun_out/sanitizer_r2/racecheck_asym.log 2>&1
for f in gpurun_out/sanitizer_r2/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $f | tail -3; done > gpurun_out/sanitizer_r2/summary.txt
echo done
