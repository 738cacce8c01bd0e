#!/bin/bash
# latency configs: BERT-base bs 1 (1 and 12 layers), empty-graph floor, W8A8 bs 1, per-kernel ncu list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 300 python - > gpurun_out/lat.json 2> gpurun_out/lat.err <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
import numpy as np
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
class A: pass
a = A(); a.model = "large"; a.seq = 128; a.batch = 256
out = bench.side_measurements(q4, synth, torch, np, torch.device("cuda"), a)
print(json.dumps({k: v for k, v in out.items() if "gemm" not in k}))
PY
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lat_launches.csv \
  python scripts/probe_latency.py 12 1 > gpurun_out/lat_ncu.log 2>&1
echo done
