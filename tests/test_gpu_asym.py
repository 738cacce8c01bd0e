"""GPU parity of the asymmetric-activation path through the C ABI
against oracle O-15 / O-16: codes, scales, zeros and INT32 bit-exact, fp16 within the
north_star tolerance."""
import numpy as np
import pytest
import torch

import oracle as orc
from paper_2301_12017_b200 import synth

pytestmark = pytest.mark.gpu


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


def rows_with_edges(M, K, name):
    x = synth.hidden(M, K, name) + np.float16(0.75)
    e = np.zeros((5, K), np.float32)
    e[0] = 3.0                                    # constant row
    e[1] = np.resize([-1.0, 0.5, 2.0], K)         # exact ties (5 (x + 1))
    e[2, 0], e[2, 1:] = 1000.0, 1e-3              # huge spread
    e[3] = np.resize([6e-8, -1.2e-7, 3e-8], K)    # subnormals
    e[4] = np.linspace(-65504, 65504, K)
    return np.concatenate([x, e.astype(np.float16)])


@pytest.mark.parametrize("rows,cols", [(1, 768), (129, 1024), (300, 4096), (3, 64)])
def test_quantize_rows_asym_bit_exact(q4, rows, cols):
    x = rows_with_edges(rows, cols, f"tas{rows}_{cols}")
    c, s, z = q4.quantize_rows_asym(dev(x))
    rc, rs, rz = orc.quantize_rows_asym(x)
    assert np.array_equal(host(c), rc)
    assert np.array_equal(host(s), rs)
    assert np.array_equal(host(z), rz)


@pytest.mark.parametrize("M,N,K", [(1, 768, 768), (129, 2304, 768), (300, 1024, 4096), (1029, 4096, 1024)])
@pytest.mark.parametrize("w8", [False, True])
def test_w4a4_asym_linear(q4, M, N, K, w8):
    x = synth.hidden(M, K, f"tal{M}_{K}") + np.float16(0.5)
    wt, b = synth.weight(N, K, f"talw{N}_{K}"), synth.bias(N, f"talb{N}")
    a, sa, za = orc.quantize_rows_asym(x)
    w, sw = orc.quantize_rows(wt)
    wd = dev(w)
    ws = q4.weight_code_sums(wd)
    assert np.array_equal(host(ws), orc.unpack_int4(w, K).astype(np.int64).sum(1).astype(np.float32))
    kw = {"w_i8": q4.prepack_weights(wd)} if w8 else {}
    i32 = q4.w4a4_asym_linear(dev(a), dev(sa), dev(za), wd, dev(sw), ws, q4.EPI_I32, **kw)["i32"]
    assert np.array_equal(host(i32), orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_I32)["i32"])
    out = q4.w4a4_asym_linear(dev(a), dev(sa), dev(za), wd, dev(sw), ws, q4.EPI_F16, bias=dev(b), **kw)["f16"]
    ref = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_F16, bias=b)["f16"]
    g, r = host(out).astype(np.float64), ref.astype(np.float64)
    assert (np.abs(g - r) <= 1e-3 + 2e-3 * np.abs(r)).all()


def test_w4a4_asym_linear_cta_pair(q4):
    """M % 256 == 0, M >= 8192, prepacked weights: the asymmetric GEMM on the CTA-pair mainloop
    (u8 x s8 with M = 256); sampled row slices against O-16."""
    M, N, K = 8192, 1024, 1024
    x = synth.hidden(M, K, "tap_x") + np.float16(0.5)
    wt, b = synth.weight(N, K, "tap_w"), synth.bias(N, "tap_b")
    a, sa, za = orc.quantize_rows_asym(x)
    w, sw = orc.quantize_rows(wt)
    wd = dev(w)
    ws = q4.weight_code_sums(wd)
    kw = {"w_i8": q4.prepack_weights(wd)}
    i32 = host(q4.w4a4_asym_linear(dev(a), dev(sa), dev(za), wd, dev(sw), ws, q4.EPI_I32, **kw)["i32"])
    f16 = host(q4.w4a4_asym_linear(dev(a), dev(sa), dev(za), wd, dev(sw), ws, q4.EPI_F16, bias=dev(b), **kw)["f16"])
    for m0 in (0, 128, M - 128):
        rows = slice(m0, m0 + 128)
        assert np.array_equal(i32[rows], orc.w4a4_asym_linear(a[rows], sa[rows], za[rows], w, sw, 128, N, K,
                                                               orc.EPI_I32)["i32"])
        r = orc.w4a4_asym_linear(a[rows], sa[rows], za[rows], w, sw, 128, N, K, orc.EPI_F16, bias=b)["f16"]
        g = f16[rows].astype(np.float64)
        assert (np.abs(g - r) <= 1e-3 + 2e-3 * np.abs(r.astype(np.float64))).all()
