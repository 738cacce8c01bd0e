"""BASELINE configs[4]: W4A4 GEMM shape sweep, M in {128..32768} x (K, N) in
{(768,3072), (3072,768), (1024,4096), (4096,1024)}, F16 (dequant + bias) epilogue, CUDA-event
timing of a CUDA graph of 20 back-to-back launches (inputs resident; the graph removes the
host launch cost that would otherwise dominate at small M), for the tcgen05 mainloop with packed
weights, with prepacked int8 weights (W8), the legacy mma.sync s8 baseline, and the W8A8
baseline (int8 activations and weights, both TMA'd into the MMA stage).  TOPS =
2*M*N*K / t; roofline = min(INT8 burst peak, HBM * ops/bytes) with the peaks of bench.peaks()
(burst: every GEMM here runs alone, not inside the long step).
Writes one JSON object per line (profiles/<round>/gemm_sweep.jsonl when run by the round script)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
from bench import peaks

pk = peaks()
int8_peak, hbm = pk["int8_tops_burst"], pk["hbm_gbs"]  # each GEMM is timed alone: burst peak
dev = torch.device("cuda")
for (K, N) in ((768, 3072), (3072, 768), (1024, 4096), (4096, 1024)):
    w = torch.from_numpy(synth.random_packed(N, K, "sw%d" % N)).to(dev)
    sw = torch.from_numpy(synth.random_scales(N, "ssw%d" % N)).to(dev)
    w8 = q4.prepack_weights(w)
    wq8 = torch.from_numpy(synth.random_i8(N, K, "sw8_%d" % N)).to(dev)
    for M in (128, 512, 2048, 8192, 12288, 32768):
        a = torch.from_numpy(synth.random_packed(M, K, "sa%d" % M)).to(dev)
        a8 = torch.from_numpy(synth.random_i8(M, K, "sa8_%d" % M)).to(dev)
        sa = torch.from_numpy(synth.random_scales(M, "ssa%d" % M)).to(dev)
        ops = 2.0 * M * N * K
        for name, ml, kw in (("tcgen05", 1, {}), ("tcgen05_w8", 4, {"w_i8": w8}), ("mma_sync_s8", 2, {}),
                             ("w8a8_tcgen05", -1, {})):
            ws = torch.zeros(max(1, q4.lib().q4_w4a4_linear_workspace(M, N, K, q4.EPI_F16)), dtype=torch.uint8,
                             device=dev)
            if ml < 0:
                def run(out=None):
                    return q4.w8a8_linear(a8, sa, wq8, sw, q4.EPI_F16, out=out, workspace=ws)
            else:
                def run(out=None, ml=ml, kw=kw):
                    return q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, mainloop=ml, out=out, workspace=ws, **kw)
            o = run()
            for _ in range(3):
                run(o)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    run(o)
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 100 * 1e-3
            wbytes = N * K if ml in (4, -1) else N * K / 2
            byt = (M * K if ml < 0 else M * K / 2) + wbytes + 4 * M + 6 * N + 2 * M * N
            roof = min(int8_peak, hbm * 1e9 * ops / byt / 1e12)
            print(json.dumps({"M": M, "N": N, "K": K, "mainloop": name, "us": round(t * 1e6, 2),
                              "TOPS": round(ops / t / 1e12, 1), "frac_int8_peak": round(ops / t / 1e12 / int8_peak, 3),
                              "roofline_TOPS": round(roof, 1), "frac_roofline": round(ops / t / 1e12 / roof, 3)}),
                  flush=True)
