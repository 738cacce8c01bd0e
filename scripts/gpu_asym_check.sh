#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_asym.py -m gpu -q -x -p no:cacheprovider > gpurun_out/asym2.log 2>&1
echo "rc=$?" >> gpurun_out/asym2.log
timeout -s KILL 300 python - >> gpurun_out/asym2.log 2>&1 <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
for asym in (False, True):
    c = dict(synth.BERT["large"])
    enc = q4.W4A4Encoder(c, [synth.layer_params(c, l, "bert") for l in range(24)], asym=asym)
    x = torch.from_numpy(np.concatenate([synth.hidden(128, 1024, "input", b) for b in range(256)])).cuda()
    o = torch.empty_like(x)
    enc.capture(x, o, 256, 128)
    for _ in range(3): enc.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(10): enc.replay()
    b.record(); torch.cuda.synchronize()
    print("asym" if asym else "sym", 256 / (a.elapsed_time(b) / 10e3), "seq/s")
PY
echo done
