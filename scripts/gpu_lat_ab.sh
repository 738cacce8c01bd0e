#!/bin/bash
# latency-config A/B (profiling build knobs): split-K, attention cluster size, W8A8; warm and
# cold per-kernel launch lists of the 12-layer BERT-base bs-1 forward.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${1:-split_k or small or layer or drift or linear or attention}" > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/ab_tests.log
P=$PWD/paper_2301_12017_b200/libq4_prof.so
run() {  # name, env...
  local name=$1; shift
  env Q4_LIB_PATH=$P "$@" timeout -s KILL 120 python scripts/probe_latency.py 12 1 > gpurun_out/ab_$name.json 2>&1
  env Q4_LIB_PATH=$P "$@" timeout -s KILL 120 python scripts/probe_latency_w8.py 12 > gpurun_out/ab_w8_$name.json 2>&1
}
run default X=1
run ksoff Q4_KSPLIT=0
run ks4 Q4_KSPLIT=4
run ks8 Q4_KSPLIT=8
run ks12 Q4_KSPLIT=12
run g12 Q4_ATTN_G=12
run g12x Q4_ATTN_G=12 Q4_ATTN_SMEM_EXTRA=20000
run g4 Q4_ATTN_G=4
run g6x Q4_ATTN_SMEM_EXTRA=20000
for f in gpurun_out/ab_*.json; do echo "$f $(tail -1 $f)"; done > gpurun_out/ab_summary.txt
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/ab_launches_warm.csv \
  python scripts/probe_latency.py 12 1 > gpurun_out/ab_ncu.log 2>&1
Q4_LIB_PATH=$P Q4_ATTN_G=12 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/ab_launches_warm_g12.csv \
  python scripts/probe_latency.py 12 1 > gpurun_out/ab_ncu2.log 2>&1
echo done
