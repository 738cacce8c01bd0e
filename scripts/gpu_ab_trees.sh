#!/bin/bash
# A/B of the current tree against the previous build copied under _abold/ (same box, interleaved)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/ab_trees.jsonl
for rep in 1 2; do
for tree in . _abold; do
  echo "== $tree" >> gpurun_out/ab_trees.jsonl
  for args in "32768 4096 1024 2 4" "32768 1024 1024 3 4" "32768 1024 4096 3 4"; do
    (cd $tree && timeout -s KILL 60 python scripts/probe_gemm.py $args) >> gpurun_out/ab_trees.jsonl 2>&1
  done
  (cd $tree && timeout -s KILL 60 python scripts/probe_attn.py) >> gpurun_out/ab_trees.jsonl 2>&1
  (cd $tree && timeout -s KILL 60 python scripts/probe_latency.py 12 1) >> gpurun_out/ab_trees.jsonl 2>&1
done
done
echo done
