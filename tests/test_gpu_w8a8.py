"""GPU parity of the W8A8 baseline through the C ABI against the
W8A8 oracle (O-11..O-13) on the same seeded inputs.  Bars as for W4A4: int8 codes,
scales and INT32 accumulators bit-exact; fp16 within |gpu - ref| <= 1e-3 + 2e-3 |ref|;
requant codes decided from the GPU's own fp16 (R13)."""
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


def assert_f16_close(got, ref, what=""):
    g, r = got.astype(np.float64), ref.astype(np.float64)
    err = np.abs(g - r) - (ATOL + RTOL * np.abs(r))
    bad = np.argwhere(err > 0)
    assert bad.size == 0, f"{what}: {len(bad)} out of tolerance, first {bad[:3].tolist()}"


def edge_rows(cols):
    z = np.zeros((6, cols), np.float32)
    z[1, 3] = 40.0
    z[1, 5:] = 0.01
    z[2, :] = np.resize([127.0, 2.5, -2.5, 0.5, -0.5, 1.5, -1.5, 126.5], cols)  # exact ties at 8 bits
    z[3, :] = np.resize([3.0, -3.0], cols)
    z[4, :] = np.resize([6e-8, -1.2e-7, 3e-8], cols)
    z[5, :] = 65504.0
    return z.astype(np.float16)


@pytest.mark.parametrize("rows,cols", [(1, 768), (129, 3072), (513, 4096), (64, 8192), (3, 64)])
def test_quantize_rows_i8_bit_exact(q4, rows, cols):
    x = np.concatenate([synth.hidden(rows, cols, f"t8q{rows}_{cols}"), edge_rows(cols)])
    c, s = q4.quantize_rows_i8(dev(x))
    rc, rs = orc.quantize_rows_i8(x)
    assert np.array_equal(host(c), rc)
    assert np.array_equal(host(s), rs)
    c, s = q4.quantize_rows_i8(dev(x), clip=5.0)
    rc, rs = orc.quantize_rows_i8(x, clip=5.0)
    assert np.array_equal(host(c), rc) and np.array_equal(host(s), rs)


@pytest.mark.parametrize("M,N,K", [(1, 768, 768), (129, 2304, 768), (300, 1024, 4096), (1029, 3072, 1024)])
def test_w8a8_i32_and_f16(q4, M, N, K):
    x, wt, b = synth.hidden(M, K, f"w8x{M}"), synth.weight(N, K, f"w8w{N}_{K}"), synth.bias(N, f"w8b{N}")
    a, sa = orc.quantize_rows_i8(x)
    w, sw = orc.quantize_rows_i8(wt)
    i32 = q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_I32)["i32"]
    assert np.array_equal(host(i32), orc.gemm_i32_i8(a, w, M, N, K))
    out = q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_F16, bias=dev(b))
    ref = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_F16, bias=b)["f16"]
    assert_f16_close(host(out["f16"]), ref, "W8A8 F16")


def test_w8a8_i32_extremes(q4):
    """all -128 operands: |acc| = 2^14 K, the largest the int8 GEMM can produce."""
    M, N, K = 130, 256, 8192
    a = np.full((M, K), -128, np.int8)
    w = np.full((N, K), -128, np.int8)
    w[1::2] = 127
    s1 = np.ones(M, np.float32)
    i32 = q4.w8a8_linear(dev(a), dev(s1), dev(w), dev(np.ones(N, np.float32)), q4.EPI_I32)["i32"]
    assert np.array_equal(host(i32), orc.gemm_i32_i8(a, w, M, N, K))


@pytest.mark.parametrize("M,N,K", [(128, 3072, 768), (1029, 4096, 1024), (33, 768, 768)])
def test_w8a8_gelu_q(q4, M, N, K):
    x, wt, b = synth.hidden(M, K, f"w8gx{M}"), synth.weight(N, K, f"w8gw{N}_{K}"), synth.bias(N, f"w8gb{N}")
    a, sa = orc.quantize_rows_i8(x)
    w, sw = orc.quantize_rows_i8(wt)
    out = q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_GELU_Q4, bias=dev(b), f16_tap=True)
    ref = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_GELU_Q4, bias=b)
    y = host(out["f16"])
    assert_f16_close(y, ref["f16"], "W8A8 GELU f16")
    c2, s2 = orc.quantize_rows_i8(y)
    assert np.array_equal(host(out["codes"]), c2)
    assert np.array_equal(host(out["scales"]), s2)
    o2 = q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_GELU_Q4, bias=dev(b))
    assert np.array_equal(host(o2["codes"]), c2)


@pytest.mark.parametrize("M,N,K", [(128, 768, 768), (1029, 1024, 4096), (7, 256, 512)])
def test_w8a8_resln_q(q4, M, N, K):
    x, wt, b = synth.hidden(M, K, f"w8lx{M}"), synth.weight(N, K, f"w8lw{N}_{K}"), synth.bias(N, f"w8lb{N}")
    res = synth.hidden(M, N, f"w8lr{M}_{N}")
    gam, bet = synth.ln_params(N, f"w8ln{N}")
    a, sa = orc.quantize_rows_i8(x)
    w, sw = orc.quantize_rows_i8(wt)
    out = q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_RESLN_Q4, bias=dev(b), residual=dev(res),
                         gamma=dev(gam), beta=dev(bet))
    ref = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res, gamma=gam, beta=bet)
    y = host(out["f16"])
    assert_f16_close(y, ref["f16"], "W8A8 RESLN f16")
    c2, s2 = orc.quantize_rows_i8(y)
    assert np.array_equal(host(out["codes"]), c2)
    assert np.array_equal(host(out["scales"]), s2)


def test_w8a8_errors(q4):
    a = torch.zeros(4, 96, dtype=torch.int8, device="cuda")  # K % 128 != 0
    s = torch.ones(4, dtype=torch.float32, device="cuda")
    w = torch.zeros(64, 96, dtype=torch.int8, device="cuda")
    with pytest.raises(Exception, match="multiple of 128"):
        q4.w8a8_linear(a, s, w, torch.ones(64, dtype=torch.float32, device="cuda"), q4.EPI_F16)
