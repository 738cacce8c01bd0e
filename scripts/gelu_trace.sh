cd $GRAFT_REPO_ROOT
rm -f /tmp/tr.bin; Q4_TRACE=/tmp/tr.bin python scripts/probe_gemm.py 32768 4096 1024 2 4 > /dev/null; python scripts/trace_gelu.py /tmp/tr.bin | tail -1; python scripts/trace_report.py /tmp/tr.bin | grep "mma\|unpack" | tail -2; python scripts/probe_gemm.py 32768 4096 1024 2 4
