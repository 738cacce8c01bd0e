"""Profiling / bring-up check of the CTA-pair mainloop (run with Q4_PAIR=1): I32 / F16 /
RESLN_Q4 GEMMs at M % 256 == 0 against the oracle (I32 exact) and the 1-CTA path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as orc
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 3072, 1024)
x, wt = synth.hidden(M, K, "pc_x"), synth.weight(N, K, "pc_w")
a, sa = orc.quantize_rows(x)
w, sw = orc.quantize_rows(wt)
wd = torch.from_numpy(w).cuda()
w8 = q4.prepack_weights(wd)
ad, sad, swd = (torch.from_numpy(t).cuda() for t in (a, sa, sw))
i32 = q4.w4a4_linear(ad, sad, wd, swd, q4.EPI_I32, w_i8=w8)["i32"]
torch.cuda.synchronize()
ref = orc.gemm_i32(a[:512], w, 512, N, K)
print("I32 rows 0..511 exact:", np.array_equal(i32[:512].cpu().numpy(), ref))
ref2 = orc.gemm_i32(a[-256:], w, 256, N, K)
print("I32 last 256 rows exact:", np.array_equal(i32[-256:].cpu().numpy(), ref2))
