#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f /tmp/at1.bin
Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_TRACE=/tmp/at1.bin timeout -s KILL 120 python scripts/probe_attn.py 1 128 12 > gpurun_out/attn1_trace.txt 2>&1
python scripts/trace_attn_bs1.py /tmp/at1.bin 12 >> gpurun_out/attn1_trace.txt 2>&1
echo done
