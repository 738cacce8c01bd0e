#!/bin/bash
# trace stamps of the FFN1 GELU_Q4 epilogue (profiling lib), per knob setting
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
rm -f gpurun_out/tr_*.bin gpurun_out/tr_report.txt
for k in ${KNOBS:-0 768}; do
  Q4_LIB_PATH=$PWD/paper_2301_12017_b200/libq4_prof.so Q4_DEBUG_SKIP=$k Q4_TRACE=/tmp/tr_$k.bin timeout -s KILL 120 \
    python scripts/probe_gemm.py ${SHAPE:-32768 4096 1024 2 4} >> gpurun_out/tr_report.txt 2>&1
  python - /tmp/tr_$k.bin >> gpurun_out/tr_report.txt 2>&1 <<'PY'
import sys, numpy as np
raw = open(sys.argv[1], "rb").read(); rec = 16 + 148*64*8*8; n = len(raw)//rec
open("/tmp/last.bin","wb").write(raw[(n-1)*rec:n*rec])
PY
  echo "== knob $k" >> gpurun_out/tr_report.txt
  python scripts/trace_report.py /tmp/last.bin >> gpurun_out/tr_report.txt 2>&1
done
echo done
