"""Bring-up: run the layer GEMM kinds at M % 256 == 0 and save outputs (compare Q4_PAIR=0/1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as orc
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
out = {}
M = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
for (N, K, kind) in ((3072, 1024, q4.EPI_F16), (1024, 1024, q4.EPI_RESLN_Q4), (1024, 4096, q4.EPI_RESLN_Q4),
                     (3072, 1024, q4.EPI_I32), (1024, 4096, q4.EPI_I32)):
    x, wt = synth.hidden(M, K, f"pcx{K}"), synth.weight(N, K, f"pcw{N}_{K}")
    a, sa = orc.quantize_rows(x)
    w, sw = orc.quantize_rows(wt)
    wd = torch.from_numpy(w).cuda()
    kw = dict(w_i8=q4.prepack_weights(wd))
    if kind == q4.EPI_RESLN_Q4:
        kw.update(residual=torch.from_numpy(synth.hidden(M, N, "pcr")).cuda(),
                  gamma=torch.ones(N, dtype=torch.float16, device="cuda"), beta=torch.zeros(N, dtype=torch.float16, device="cuda"))
    o = q4.w4a4_linear(torch.from_numpy(a).cuda(), torch.from_numpy(sa).cuda(), wd, torch.from_numpy(sw).cuda(), kind, **kw)
    torch.cuda.synchronize()
    for k, v in o.items():
        out[f"{N}_{K}_{kind}_{k}"] = v.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", len(out))
