#!/bin/bash
# round-2 profile evidence: launch list + one-layer full capture (profile_round.sh) + GEMM sweep
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash scripts/profile_round.sh r2
timeout -s KILL 900 python scripts/gemm_sweep.py > gpurun_out/r2_gemm_sweep.jsonl 2> gpurun_out/r2_gemm_sweep.err
echo done
