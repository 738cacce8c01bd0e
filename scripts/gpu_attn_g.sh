#!/bin/bash
# attention at B=256: cluster split G (profiling lib, Q4_ATTN_G) A/B
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/attn_g.jsonl
timeout -s KILL 120 python scripts/probe_attn.py >> gpurun_out/attn_g.jsonl 2>&1
for g in 1 2 4 8; do
  echo "G=$g" >> gpurun_out/attn_g.jsonl
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_ATTN_G=$g timeout -s KILL 120 python scripts/probe_attn.py >> gpurun_out/attn_g.jsonl 2>&1
done
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "attention" > gpurun_out/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/attn_tests.log
echo done
