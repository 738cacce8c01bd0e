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


# ------------------------------------------------------------------ a7 / a8 at 8 bits
@pytest.mark.parametrize("B,S,H", [(2, 128, 12), (3, 128, 16), (1, 77, 16), (4, 1, 2)])
def test_attention_q8(q4, B, S, H):
    qkv = synth.hidden(B * S, 3 * H * 64, f"a8q{B}_{S}_{H}")
    codes, scales, ctx = q4.attention_f16_q8(dev(qkv), B, S, H, 64, f16_tap=True)
    rctx, _, _ = orc.attention(qkv, B, S, H, 64)
    c = host(ctx)
    assert_f16_close(c, rctx, "ctx")
    c2, s2 = orc.quantize_rows_i8(c)  # O-11 on the GPU's own fp16 ctx (R13)
    assert np.array_equal(host(codes), c2) and np.array_equal(host(scales), s2)


@pytest.mark.parametrize("size,B", [("base", 2), ("large", 1)])
def test_encoder_layer_w8a8_teacher_forced(q4, size, B):
    """Every sub-step of q4_encoder_layer_w8a8 against the W8A8 oracle on the GPU's own
    inputs (taps): INT32 bit-exact, fp16 within tolerance, codes = O-11(GPU fp16)."""
    cfg = synth.BERT[size]
    S, M, h, f = 128, B * 128, cfg["hidden"], cfg["ffn"]
    p = synth.layer_params(cfg, 0, "enc8")
    x = synth.hidden(M, h, "enc8_x")
    w = q4.quantize_layer(p, bits=8)
    for k in ("wqkv", "wo", "w1", "w2"):
        rc, rs = orc.quantize_rows_i8(p[k])
        assert np.array_equal(host(w[k]), rc) and np.array_equal(host(w["s" + k[1:]]), rs), k
    xq, xs = q4.quantize_rows_i8(dev(x))
    out = q4.encoder_layer(cfg, w, B, S, dev(x), xq, xs, taps=True, bits=8)
    T = {k: host(v) for k, v in out.items()}
    W = {k: host(v) for k, v in w.items()}
    xq_, xs_ = host(xq), host(xs)
    assert np.array_equal(T["acc_qkv"], orc.gemm_i32_i8(xq_, W["wqkv"], M, 3 * h, h))
    rq = orc.w8a8_linear(xq_, xs_, W["wqkv"], W["sqkv"], M, 3 * h, h, orc.EPI_F16, bias=p["bqkv"])
    assert_f16_close(T["qkv"], rq["f16"], "qkv")
    rctx, _, _ = orc.attention(T["qkv"], B, S, cfg["heads"], 64)
    assert_f16_close(T["ctx"], rctx, "ctx")
    c2, s2 = orc.quantize_rows_i8(T["ctx"])
    assert np.array_equal(T["ctx_codes"], c2) and np.array_equal(T["ctx_scales"], s2)
    assert np.array_equal(T["acc_o"], orc.gemm_i32_i8(T["ctx_codes"], W["wo"], M, h, h))
    r1 = orc.w8a8_linear(T["ctx_codes"], T["ctx_scales"], W["wo"], W["so"], M, h, h, orc.EPI_RESLN_Q4,
                         bias=p["bo"], residual=x, gamma=p["ln1_g"], beta=p["ln1_b"])
    assert_f16_close(T["h1"], r1["f16"], "h1")
    c2, s2 = orc.quantize_rows_i8(T["h1"])
    assert np.array_equal(T["h1_codes"], c2) and np.array_equal(T["h1_scales"], s2)
    assert np.array_equal(T["acc_1"], orc.gemm_i32_i8(T["h1_codes"], W["w1"], M, f, h))
    r2 = orc.w8a8_linear(T["h1_codes"], T["h1_scales"], W["w1"], W["s1"], M, f, h, orc.EPI_GELU_Q4, bias=p["b1"])
    assert_f16_close(T["ffn1"], r2["f16"], "ffn1")
    c2, s2 = orc.quantize_rows_i8(T["ffn1"])
    assert np.array_equal(T["f_codes"], c2) and np.array_equal(T["f_scales"], s2)
    assert np.array_equal(T["acc_2"], orc.gemm_i32_i8(T["f_codes"], W["w2"], M, h, f))
    r3 = orc.w8a8_linear(T["f_codes"], T["f_scales"], W["w2"], W["s2"], M, h, f, orc.EPI_RESLN_Q4,
                         bias=p["b2"], residual=T["h1"], gamma=p["ln2_g"], beta=p["ln2_b"])
    assert_f16_close(T["h_out"], r3["f16"], "h_out")
    c2, s2 = orc.quantize_rows_i8(T["h_out"])
    assert np.array_equal(T["hq_out"], c2) and np.array_equal(T["hs_out"], s2)


def test_encoder_stack_w8a8_host_device_graph(q4):
    """The W8A8 stack: device call == host-buffer (end-to-end) call == CUDA-graph replay,
    and layer 0 of the stack equals q4_encoder_layer_w8a8 on the same input."""
    cfg = synth.BERT["base"]
    B, S, L = 2, 128, 3
    layers = [synth.layer_params(cfg, l, "stk8") for l in range(L)]
    x = synth.hidden(B * S, cfg["hidden"], "stk8_x")
    enc = q4.W8A8Encoder(cfg, layers)
    xd = dev(x)
    o1 = torch.empty_like(xd)
    enc.forward(xd, o1, B, S)
    oh = torch.empty(xd.shape, dtype=torch.float16).pin_memory()
    enc.forward(torch.from_numpy(x).pin_memory(), oh, B, S)
    torch.cuda.synchronize()
    assert torch.equal(oh, o1.cpu())
    o2 = torch.empty_like(xd)
    enc.capture(xd, o2, B, S)
    enc.replay()
    assert torch.equal(o2, o1)
    one = q4.W8A8Encoder(cfg, layers[:1])
    o3 = torch.empty_like(xd)
    one.forward(xd, o3, B, S)
    xq, xs = q4.quantize_rows_i8(xd)
    ref = q4.encoder_layer(cfg, one.weights[0], B, S, xd, xq, xs, bits=8)
    assert torch.equal(o3, ref["h_out"])


# ------------------------------------------------------------------ NEXT-1: FP16 parts
@pytest.mark.parametrize("M,N,K", [(1, 768, 768), (129, 2304, 768), (300, 1024, 4096), (1029, 4096, 1024)])
def test_f16_linear(q4, M, N, K):
    """The FP16 tcgen05 GEMM (kind::f16, fp32 accumulate) with the fused epilogues against
    O-14; INT4 codes decided from the GPU's own fp16 (R13)."""
    a, w, b = synth.hidden(M, K, f"h16a{M}"), synth.weight(N, K, f"h16w{N}_{K}"), synth.bias(N, f"h16b{N}")
    out = q4.f16_linear(dev(a), dev(w), q4.EPI_F16, bias=dev(b))
    ref = orc.f16_linear(a, w, M, N, K, orc.EPI_F16, bias=b)["f16"]
    assert_f16_close(host(out["f16"]), ref, "F16 linear")
    out = q4.f16_linear(dev(a), dev(w), q4.EPI_GELU_Q4, bias=dev(b), f16_tap=True)
    ref = orc.f16_linear(a, w, M, N, K, orc.EPI_GELU_Q4, bias=b)
    y = host(out["f16"])
    assert_f16_close(y, ref["f16"], "F16 linear GELU")
    c2, s2 = orc.quantize_rows(y)
    assert np.array_equal(host(out["codes"]), c2) and np.array_equal(host(out["scales"]), s2)
    if N <= 1024:
        res = synth.hidden(M, N, f"h16r{M}")
        gam, bet = synth.ln_params(N, f"h16ln{N}")
        out = q4.f16_linear(dev(a), dev(w), q4.EPI_RESLN_Q4, bias=dev(b), residual=dev(res), gamma=dev(gam),
                            beta=dev(bet))
        ref = orc.f16_linear(a, w, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res, gamma=gam, beta=bet)
        y = host(out["f16"])
        assert_f16_close(y, ref["f16"], "F16 linear RESLN")
        c2, s2 = orc.quantize_rows(y)
        assert np.array_equal(host(out["codes"]), c2) and np.array_equal(host(out["scales"]), s2)


@pytest.mark.parametrize("fp16_parts", [0xB, 0x4, 0xF, 0x6])
def test_encoder_layer_strategy_teacher_forced(q4, fp16_parts):
    """Per-part quantization strategy: each part runs W4A4 or FP16 as the
    mask says; every sub-step checked on the GPU's own inputs against O-5..O-8 / O-14."""
    cfg = dict(synth.BERT["base"], fp16_parts=fp16_parts)
    B, S = 2, 128
    M, h, f = B * S, cfg["hidden"], cfg["ffn"]
    p = synth.layer_params(cfg, 0, "encs")
    x = synth.hidden(M, h, "encs_x")
    w = q4.quantize_layer(p, fp16_parts=fp16_parts)
    xq, xs = q4.quantize_rows(dev(x))
    out = q4.encoder_layer(cfg, w, B, S, dev(x), xq, xs, taps=True)
    T = {k: host(v) for k, v in out.items()}
    W = {k: host(v) for k, v in w.items()}

    def part(i, a16, codes, scales, wname, N, K, epi, **kw):
        if fp16_parts >> i & 1:
            return orc.f16_linear(a16, p["w" + wname], M, N, K, epi, **kw)
        return orc.w4a4_linear(codes, scales, W["w" + wname], W["s" + wname], M, N, K, epi, **kw)

    rq = part(0, x, host(xq), host(xs), "qkv", 3 * h, h, orc.EPI_F16, bias=p["bqkv"])
    assert_f16_close(T["qkv"], rq["f16"], "qkv")
    rctx, _, _ = orc.attention(T["qkv"], B, S, cfg["heads"], 64)
    assert_f16_close(T["ctx"], rctx, "ctx")
    r1 = part(1, T["ctx"], T["ctx_codes"], T["ctx_scales"], "o", h, h, orc.EPI_RESLN_Q4, bias=p["bo"],
              residual=x, gamma=p["ln1_g"], beta=p["ln1_b"])
    assert_f16_close(T["h1"], r1["f16"], "h1")
    c2, s2 = orc.quantize_rows(T["h1"])
    assert np.array_equal(T["h1_codes"], c2) and np.array_equal(T["h1_scales"], s2)
    r2 = part(2, T["h1"], T["h1_codes"], T["h1_scales"], "1", f, h, orc.EPI_GELU_Q4, bias=p["b1"])
    assert_f16_close(T["ffn1"], r2["f16"], "ffn1")
    c2, s2 = orc.quantize_rows(T["ffn1"])
    assert np.array_equal(T["f_codes"], c2) and np.array_equal(T["f_scales"], s2)
    r3 = part(3, T["ffn1"], T["f_codes"], T["f_scales"], "2", h, f, orc.EPI_RESLN_Q4, bias=p["b2"],
              residual=T["h1"], gamma=p["ln2_g"], beta=p["ln2_b"])
    assert_f16_close(T["h_out"], r3["f16"], "h_out")


def test_encoder_stack_strategy_graph(q4):
    """q3-only strategy (0xB): device call == host-buffer call == graph replay."""
    cfg = synth.BERT["base"]
    B, S, L = 1, 128, 2
    layers = [synth.layer_params(cfg, l, "stks") for l in range(L)]
    x = synth.hidden(B * S, cfg["hidden"], "stks_x")
    enc = q4.W4A4Encoder(cfg, layers, fp16_parts=0xB)
    xd = dev(x)
    o1 = torch.empty_like(xd)
    enc.forward(xd, o1, B, S)
    oh = torch.empty(xd.shape, dtype=torch.float16).pin_memory()
    enc.forward(torch.from_numpy(x).pin_memory(), oh, B, S)
    torch.cuda.synchronize()
    assert torch.equal(oh, o1.cpu())
    o2 = torch.empty_like(xd)
    enc.capture(xd, o2, B, S)
    enc.replay()
    assert torch.equal(o2, o1)


def test_w8a8_full_size_layer_sampled(q4):
    """The W8A8 baseline at the bench's launch configuration (BERT-large, M = 32768): sampled
    sequences checked teacher-forced against the W8A8 oracle (independent sub-problems)."""
    cfg = synth.BERT["large"]
    B, S = 256, 128
    M, h, f = B * S, cfg["hidden"], cfg["ffn"]
    p = synth.layer_params(cfg, 0, "full8")
    x = synth.hidden(M, h, "full8_x")
    w = q4.quantize_layer(p, bits=8)
    xq, xs = q4.quantize_rows_i8(dev(x))
    out = q4.encoder_layer(cfg, w, B, S, dev(x), xq, xs, taps=True, bits=8)
    torch.cuda.synchronize()
    W = {k: host(v) for k, v in w.items()}
    for bsel in (0, 201, 255):
        rows = slice(bsel * S, (bsel + 1) * S)
        T = {k: host(v[rows]) for k, v in out.items()}
        xq_, xs_ = host(xq[rows]), host(xs[rows])
        assert np.array_equal(T["acc_qkv"], orc.gemm_i32_i8(xq_, W["wqkv"], S, 3 * h, h))
        rctx, _, _ = orc.attention(T["qkv"], 1, S, cfg["heads"], 64)
        assert_f16_close(T["ctx"], rctx, "ctx")
        c2, s2 = orc.quantize_rows_i8(T["ctx"])
        assert np.array_equal(T["ctx_codes"], c2) and np.array_equal(T["ctx_scales"], s2)
        assert np.array_equal(T["acc_o"], orc.gemm_i32_i8(T["ctx_codes"], W["wo"], S, h, h))
        assert np.array_equal(T["acc_1"], orc.gemm_i32_i8(T["h1_codes"], W["w1"], S, f, h))
        r2 = orc.w8a8_linear(T["h1_codes"], T["h1_scales"], W["w1"], W["s1"], S, f, h, orc.EPI_GELU_Q4, bias=p["b1"])
        assert_f16_close(T["ffn1"], r2["f16"], "ffn1")
        assert np.array_equal(T["acc_2"], orc.gemm_i32_i8(T["f_codes"], W["w2"], S, h, f))
        r3 = orc.w8a8_linear(T["f_codes"], T["f_scales"], W["w2"], W["s2"], S, h, f, orc.EPI_RESLN_Q4,
                             bias=p["b2"], residual=T["h1"], gamma=p["ln2_g"], beta=p["ln2_b"])
        assert_f16_close(T["h_out"], r3["f16"], "h_out")
        c2, s2 = orc.quantize_rows_i8(T["h_out"])
        assert np.array_equal(T["hq_out"], c2) and np.array_equal(T["hs_out"], s2)


def test_w8a8_cta_pair(q4):
    """W8A8 at M % 256 == 0, M >= 8192 runs on the CTA-pair mainloop: sampled slices exact."""
    M, N, K = 8192, 3072, 1024
    a = synth.random_i8(M, K, "w8p_a")
    w = synth.random_i8(N, K, "w8p_w")
    sa, sw = synth.random_scales(M, "w8p_sa"), synth.random_scales(N, "w8p_sw")
    i32 = host(q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_I32)["i32"])
    f16 = host(q4.w8a8_linear(dev(a), dev(sa), dev(w), dev(sw), q4.EPI_F16)["f16"])
    for m0 in (0, 128, M - 128):
        rows = slice(m0, m0 + 128)
        assert np.array_equal(i32[rows], orc.gemm_i32_i8(a[rows], w, 128, N, K)), m0
        assert_f16_close(f16[rows], orc.w8a8_linear(a[rows], sa[rows], w, sw, 128, N, K, orc.EPI_F16)["f16"], "pair")


@pytest.mark.slow
def test_quantize_i8_exhaustive_fp16_pairs(q4):
    """Every (x, amax) fp16 pair with 0 <= x <= amax through the 8-bit CUDA quantizer equals
    the exact rational rounding rhe(127 x / amax) (O-11), computed here in int64 on the
    fp16 values as integers in units of 2^-24.  (At 8 bits the IEEE-division form is not a
    valid reference: the quotient can land within half an ulp of a half-integer.)"""
    bits = np.arange(1, 0x7C00, dtype=np.uint16)
    allpos = bits.view(np.float16)
    ival = (allpos.astype(np.float64) * 2.0 ** 24).astype(np.int64)  # exact
    n = allpos.size
    chunk = 512
    for s in range(0, n, chunk):
        idx = np.arange(s, min(n, s + chunk))
        width = ((idx[-1] + 1 + 7) // 8) * 8
        X = np.zeros((idx.size, width), np.float16)
        for r, i in enumerate(idx):
            X[r, : i + 1] = allpos[: i + 1]
        c, sc = q4.quantize_rows_i8(dev(X))
        q = host(c).astype(np.int64)
        Xi = (X.astype(np.float64) * 2.0 ** 24).astype(np.int64)
        A = ival[idx][:, None]
        num, den = 254 * Xi + A, 2 * A  # rhe(127 X / A) = floor((254 X + A) / 2A), ties to even
        ref = num // den
        tie = (num % den == 0) & (ref % 2 == 1)
        ref = ref - tie
        mask = np.arange(width)[None, :] <= idx[:, None]
        assert np.array_equal(q[mask], ref[mask]), f"chunk {s}"
        assert np.array_equal(host(sc), allpos[idx].astype(np.float32) / np.float32(127))
