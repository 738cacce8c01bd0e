"""Time one W4A4 GEMM launch configuration (profiling helper; honours Q4_DEBUG_SKIP)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth

M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 4096, 1024)))
kind = int(sys.argv[4]) if len(sys.argv) > 4 else q4.EPI_F16
ml = int(sys.argv[5]) if len(sys.argv) > 5 else 1
dev = torch.device("cuda")
a = torch.from_numpy(synth.random_packed(M, K, "pa")).to(dev)
w = torch.from_numpy(synth.random_packed(N, K, "pw")).to(dev)
sa = torch.from_numpy(synth.random_scales(M, "psa")).to(dev)
sw = torch.from_numpy(synth.random_scales(N, "psw")).to(dev)
res = torch.zeros(M, N, dtype=torch.float16, device=dev)
g = torch.ones(N, dtype=torch.float16, device=dev)
kw = dict(residual=res, gamma=g, beta=g) if kind == q4.EPI_RESLN_Q4 else {}
kw["mainloop"] = ml
if ml == 4:
    kw["w_i8"] = q4.prepack_weights(w)
ws_bytes = q4.lib().q4_w4a4_linear_workspace(M, N, K, kind)
kw["workspace"] = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
o = q4.w4a4_linear(a, sa, w, sw, kind, **kw)
for _ in range(3):
    q4.w4a4_linear(a, sa, w, sw, kind, out=o, **kw)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
if os.environ.get("PROBE_GRAPH"):
    # 20 launches in one CUDA graph: no host overhead between them (short kernels)
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        q4.w4a4_linear(a, sa, w, sw, kind, out=o, **kw)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(20):
            q4.w4a4_linear(a, sa, w, sw, kind, out=o, **kw)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
else:
    e0.record()
    for _ in range(20):
        q4.w4a4_linear(a, sa, w, sw, kind, out=o, **kw)
    e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 20
print(json.dumps({"M": M, "N": N, "K": K, "kind": kind, "mainloop": ml, "skip": os.environ.get("Q4_DEBUG_SKIP", "0"),
                  "us": t * 1e3, "TOPS": 2.0 * M * N * K / (t * 1e-3) / 1e12}))
