#!/bin/bash
# Quick timing (profiling helper): full bench step without side measurements + per-kernel times.
cd $GRAFT_REPO_ROOT
python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/q.json 2>gpurun_out/q.err
python - <<'P'
import json
d=json.load(open('gpurun_out/q.json'))
print("seq/s", round(d["value"]), "ms", round(d["ms_per_step"],3))
for k,v in d["kernels"].items(): print(k, round(v["ms"]*1e3,1), "us", round(v["TOPS"]), "TOPS")
P
