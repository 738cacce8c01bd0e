"""NEXT-4 measurement: 2:4-sparse W4A4 GEMM (tcgen05.mma.sp) vs the dense W4A4 GEMM (prepacked
weights) on the BERT-large FFN shapes and the QKV shape, F16 epilogue; dense-equivalent TOPS
= 2 M N K / t (the sparse kernel does half the multiply-adds)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e-3


dev = torch.device("cuda")
for (M, N, K) in ((32768, 4096, 1024), (32768, 1024, 4096), (32768, 3072, 1024), (128, 3072, 768), (128, 768, 3072)):
    wt = torch.from_numpy(synth.weight(N, K, f"sb{N}_{K}")).to(dev)
    w, sw = q4.quantize_rows(q4.prune_24(wt))
    vals, meta, _ = q4.sparse24_compress(w)
    w8 = q4.prepack_weights(w)
    a = torch.from_numpy(synth.random_packed(M, K, f"sba{M}_{K}")).to(dev)
    sa = torch.from_numpy(synth.random_scales(M, "sbs")).to(dev)
    o = q4.w4a4_sparse24_linear(a, sa, vals, meta, sw)
    ts = timeit(lambda: q4.w4a4_sparse24_linear(a, sa, vals, meta, sw, out=o))
    od = q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, w_i8=w8)
    td = timeit(lambda: q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, w_i8=w8, out=od))
    ops = 2.0 * M * N * K
    print(json.dumps({"M": M, "N": N, "K": K, "sparse_us": ts * 1e6, "dense_us": td * 1e6,
                      "sparse_dense_equiv_TOPS": ops / ts / 1e12, "dense_TOPS": ops / td / 1e12,
                      "speedup": td / ts}), flush=True)
