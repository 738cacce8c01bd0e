"""GPU parity of the 2:4-sparse W4A4 path through the C ABI: q4_prune_24
== O-17 bit for bit; q4_w4a4_sparse24_linear (tcgen05.mma.sp) == the dense oracle O-4 / O-5 on
the pruned, quantized weights -- INT32 bit-exact, fp16 within the north_star tolerance."""
import numpy as np
import pytest
import torch

import oracle as orc
from paper_2301_12017_b200 import synth

pytestmark = pytest.mark.gpu
RTOL, ATOL = 2e-3, 1e-3


@pytest.fixture(scope="module")
def q4():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_12017_b200 as q4
    q4.lib()
    return q4


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def sparse_weights(q4, N, K, name):
    """P => Q: l1 2:4 pruning, then per-output-channel INT4 (O-3)."""
    wt = synth.weight(N, K, name)
    wp = orc.prune_24(wt)
    assert np.array_equal(host(q4.prune_24(dev(wt))), wp)  # the GPU pruning is O-17 exactly
    w, sw = orc.quantize_rows(wp)
    vals, meta, bad = q4.sparse24_compress(dev(w))
    assert int(host(bad)[0]) == 0
    return w, sw, vals, meta


@pytest.mark.parametrize("M,N,K", [(1, 128, 256), (100, 768, 768), (257, 1024, 1024), (1029, 3072, 768),
                                   (512, 1024, 4096), (640, 4096, 1024)])
def test_sparse24_linear(q4, M, N, K):
    w, sw, vals, meta = sparse_weights(q4, N, K, f"sp{N}_{K}")
    x = synth.hidden(M, K, f"spx{M}_{K}")
    a, sa = orc.quantize_rows(x)
    b = synth.bias(N, f"spb{N}")
    i32 = q4.w4a4_sparse24_linear(dev(a), dev(sa), vals, meta, dev(sw), q4.EPI_I32)["i32"]
    assert np.array_equal(host(i32), orc.gemm_i32(a, w, M, N, K))
    f16 = q4.w4a4_sparse24_linear(dev(a), dev(sa), vals, meta, dev(sw), q4.EPI_F16, bias=dev(b))["f16"]
    ref = orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_F16, bias=b)["f16"]
    g, r = host(f16).astype(np.float64), ref.astype(np.float64)
    assert (np.abs(g - r) <= ATOL + RTOL * np.abs(r)).all()


def test_sparse24_extreme_codes(q4):
    """All kept codes -8 (the INT32 bound) and groups with fewer than two nonzeros."""
    M, N, K = 130, 256, 512
    q = np.zeros((N, K), np.int8)
    q[:, 0::4] = -8
    q[:, 3::4] = -8
    q[::3, 3::4] = 0          # one nonzero in the group
    q[::5, 0::4] = 0
    w = orc.pack_int4(q)
    vals, meta, bad = q4.sparse24_compress(dev(w))
    assert int(host(bad)[0]) == 0
    a = orc.pack_int4(np.full((M, K), -8, np.int8))
    sa, sw = np.ones(M, np.float32), np.ones(N, np.float32)
    i32 = q4.w4a4_sparse24_linear(dev(a), dev(sa), vals, meta, dev(sw), q4.EPI_I32)["i32"]
    assert np.array_equal(host(i32), orc.gemm_i32(a, w, M, N, K))


def test_sparse24_compress_counts_violations(q4):
    q = np.ones((128, 256), np.int8)  # four nonzeros per group: not 2:4
    vals, meta, bad = q4.sparse24_compress(dev(orc.pack_int4(q)))
    assert int(host(bad)[0]) == 128 * 256 // 4
