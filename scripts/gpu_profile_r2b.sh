#!/bin/bash
# round-2 evidence refresh: full GPU suite, bench line, launch list + full captures, GEMM sweep,
# batch-1 warm launch list
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/p_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/p_tests.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
echo "bench rc=$?" >> gpurun_out/p_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/p_tests.log
bash scripts/profile_round.sh r2
rm -f gpurun_out/r2_ffn1.ncu-rep
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/r2_bs1_launches.csv python scripts/probe_latency.py 12 1 > gpurun_out/r2_bs1_ncu.log 2>&1
timeout -s KILL 900 python scripts/gemm_sweep.py > gpurun_out/r2_gemm_sweep.jsonl 2> gpurun_out/r2_gemm_sweep.err
du -sh gpurun_out/* | sort -h | tail -5
echo done
