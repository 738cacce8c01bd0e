#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f /tmp/at.bin
Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_TRACE=/tmp/at.bin timeout -s KILL 120 python scripts/probe_attn.py > gpurun_out/attn_trace.txt 2>&1
python scripts/trace_attn.py /tmp/at.bin 256 >> gpurun_out/attn_trace.txt 2>&1
echo done
