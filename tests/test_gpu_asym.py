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


RTOL, ATOL = 2e-3, 1e-3


def assert_f16_close(got, ref, what=""):
    g, r = got.astype(np.float64), ref.astype(np.float64)
    err = np.abs(g - r) - (ATOL + RTOL * np.abs(r))
    bad = np.argwhere(err > 0)
    assert bad.size == 0, f"{what}: {len(bad)} out of tolerance, first {bad[:3].tolist()}"


def assert_asym_codes(q4out, y, what=""):
    """codes / scales / zeros == O-15 of the GPU's own fp16 output (R13), bit for bit."""
    c, s, z = orc.quantize_rows_asym(y)
    assert np.array_equal(host(q4out["codes"]), c), what + " codes"
    assert np.array_equal(host(q4out["scales"]), s), what + " scales"
    assert np.array_equal(host(q4out["zeros"]), z), what + " zeros"


# ------------------------------------------------------------------ NEXT-3: asymmetric requant epilogues
@pytest.mark.parametrize("M,N,K", [(37, 768, 256), (640, 4096, 1024), (1029, 1024, 768)])
def test_symmetric_input_asymmetric_output(q4, M, N, K):
    """q4_w4a4_linear with epi->out_zeros: symmetric codes in, O-15 codes out (GELU_Q4 and
    RESLN_Q4; TN = 64 below M = 512, several TN = 256 tiles per CTA above)."""
    x, wt, b = synth.hidden(M, K, f"sa{M}"), synth.weight(N, K, f"sw{N}_{K}"), synth.bias(N, f"sb{N}")
    a, sa = orc.quantize_rows(x)
    w, sw = orc.quantize_rows(wt)
    wd = dev(w)
    w8 = q4.prepack_weights(wd)
    out = q4.w4a4_linear(dev(a), dev(sa), wd, dev(sw), q4.EPI_GELU_Q4, bias=dev(b), f16_tap=True, w_i8=w8,
                         asym_out=True)
    y = host(out["f16"])
    assert_f16_close(y, orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_GELU_Q4, bias=b)["f16"], "gelu")
    assert_asym_codes(out, y, "gelu")
    res = synth.hidden(M, N, f"sr{M}_{N}")
    g, bt = synth.ln_params(N, f"sln{N}")
    out = q4.w4a4_linear(dev(a), dev(sa), wd, dev(sw), q4.EPI_RESLN_Q4, bias=dev(b), residual=dev(res),
                         gamma=dev(g), beta=dev(bt), w_i8=w8, asym_out=True)
    y = host(out["f16"])
    ref = orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res, gamma=g, beta=bt)
    assert_f16_close(y, ref["f16"], "resln")
    assert_asym_codes(out, y, "resln")


@pytest.mark.parametrize("M,N,K,w8", [(33, 768, 768, False), (300, 3072, 768, True), (1029, 4096, 1024, True),
                                      (2048, 1024, 4096, True)])
@pytest.mark.parametrize("asym_out", [True, False])
def test_asym_linear_row_epilogues(q4, M, N, K, w8, asym_out):
    """q4_w4a4_asym_linear with GELU_Q4 / RESLN_Q4 (asymmetric input, zero-point term in the
    dequant) against O-16; codes from the GPU fp16 (O-15 or O-1)."""
    x = rows_with_edges(M - 5, K, f"ar{M}")[:-1]  # the +-65504 row would overflow the fp16 outputs
    x = np.concatenate([x, synth.hidden(1, K, f"ar1{M}")])
    a, sa, za = orc.quantize_rows_asym(x)
    w, sw = orc.quantize_rows(synth.weight(N, K, f"aw{N}_{K}"))
    b = synth.bias(N, f"ab{N}")
    wd = dev(w)
    sums = q4.weight_code_sums(wd)
    kw = dict(w_i8=q4.prepack_weights(wd)) if w8 else {}
    res = synth.hidden(M, N, f"arr{M}_{N}")
    g, bt = synth.ln_params(N, f"arln{N}")
    for epi, ekw, okw in ((q4.EPI_GELU_Q4, dict(f16_tap=True), {}),
                          (q4.EPI_RESLN_Q4, dict(residual=dev(res), gamma=dev(g), beta=dev(bt)),
                           dict(residual=res, gamma=g, beta=bt))):
        out = q4.w4a4_asym_linear(dev(a), dev(sa), dev(za), wd, dev(sw), sums, epi, bias=dev(b), asym_out=asym_out,
                                  **ekw, **kw)
        y = host(out["f16"])
        ref = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, epi, bias=b, asym_out=asym_out, **okw)
        assert_f16_close(y, ref["f16"], f"asym epi {epi}")
        if asym_out:
            assert_asym_codes(out, y, f"epi {epi}")
        else:
            c, s = orc.quantize_rows(y)
            assert np.array_equal(host(out["codes"]), c) and np.array_equal(host(out["scales"]), s)


@pytest.mark.parametrize("B,S,H", [(1, 128, 12), (3, 77, 16), (160, 128, 16)])
def test_attention_asym_codes(q4, B, S, H):
    """q4_attention_f16_q4_asym: ctx vs O-8, ctx codes / scales / zeros == O-15(GPU ctx) (the
    cluster tail at small B, the single-CTA tail at B >= 148)."""
    qkv = synth.hidden(B * S, 3 * H * 64, f"aq{B}_{S}")
    c, s, z, ctx = q4.attention_f16_q4_asym(dev(qkv), B, S, H)
    cx = host(ctx)
    rctx, _, _ = orc.attention(qkv, B, S, H, 64)
    assert_f16_close(cx, rctx, "ctx")
    rc, rs, rz = orc.quantize_rows_asym(cx)
    assert np.array_equal(host(c), rc) and np.array_equal(host(s), rs) and np.array_equal(host(z), rz)


@pytest.mark.parametrize("size,B", [("base", 2), ("large", 1)])
def test_asym_encoder_layer_teacher_forced(q4, size, B):
    """The asymmetric encoder layer (q4_encoder_layer_asym, cfg.asym_acts = 1), teacher-forced:
    every sub-step on the GPU's own inputs against O-16 / O-8 / O-15 (INT32 taps bit-exact)."""
    cfg = dict(synth.BERT[size])
    cfg["asym_acts"] = 1
    S, M, h, f = 128, B * 128, cfg["hidden"], cfg["ffn"]
    p = synth.layer_params(cfg, 0, "alay")
    x = synth.hidden(M, h, "alay_x")
    w = q4.quantize_layer(p, asym=True)
    W = {k: host(v) for k, v in w.items()}
    for k in ("wqkv", "wo", "w1", "w2"):  # the zero-point term's weight code sums, exact
        assert np.array_equal(W["c" + k[1:]], orc.unpack_int4(W[k], W[k].shape[1] * 2).sum(1).astype(np.float32))
    xq, xs, xz = q4.quantize_rows_asym(dev(x))
    out = q4.encoder_layer(cfg, w, B, S, dev(x), xq, xs, taps=True, hz_in=xz)
    T = {k: host(v) for k, v in out.items()}
    xq_, xs_, xz_ = host(xq), host(xs), host(xz)

    def acc_ref(codes, wc, N, K):
        qa = orc.unpack_u4(codes, K).astype(np.int64)
        return (qa @ orc.unpack_int4(wc, K).astype(np.int64).T).astype(np.int32)

    assert np.array_equal(T["acc_qkv"], acc_ref(xq_, W["wqkv"], 3 * h, h))
    rq = orc.w4a4_asym_linear(xq_, xs_, xz_, W["wqkv"], W["sqkv"], M, 3 * h, h, orc.EPI_F16, bias=p["bqkv"])
    assert_f16_close(T["qkv"], rq["f16"], "qkv")
    rctx, _, _ = orc.attention(T["qkv"], B, S, cfg["heads"], 64)
    assert_f16_close(T["ctx"], rctx, "ctx")
    c, s, z = orc.quantize_rows_asym(T["ctx"])
    assert np.array_equal(T["ctx_codes"], c) and np.array_equal(T["ctx_scales"], s) and np.array_equal(T["ctx_zeros"], z)
    assert np.array_equal(T["acc_o"], acc_ref(T["ctx_codes"], W["wo"], h, h))
    r1 = orc.w4a4_asym_linear(T["ctx_codes"], T["ctx_scales"], T["ctx_zeros"], W["wo"], W["so"], M, h, h,
                              orc.EPI_RESLN_Q4, bias=p["bo"], residual=x, gamma=p["ln1_g"], beta=p["ln1_b"])
    assert_f16_close(T["h1"], r1["f16"], "h1")
    c, s, z = orc.quantize_rows_asym(T["h1"])
    assert np.array_equal(T["h1_codes"], c) and np.array_equal(T["h1_scales"], s) and np.array_equal(T["h1_zeros"], z)
    assert np.array_equal(T["acc_1"], acc_ref(T["h1_codes"], W["w1"], f, h))
    r2 = orc.w4a4_asym_linear(T["h1_codes"], T["h1_scales"], T["h1_zeros"], W["w1"], W["s1"], M, f, h,
                              orc.EPI_GELU_Q4, bias=p["b1"])
    assert_f16_close(T["ffn1"], r2["f16"], "ffn1")
    c, s, z = orc.quantize_rows_asym(T["ffn1"])
    assert np.array_equal(T["f_codes"], c) and np.array_equal(T["f_scales"], s) and np.array_equal(T["f_zeros"], z)
    assert np.array_equal(T["acc_2"], acc_ref(T["f_codes"], W["w2"], h, f))
    r3 = orc.w4a4_asym_linear(T["f_codes"], T["f_scales"], T["f_zeros"], W["w2"], W["s2"], M, h, f,
                              orc.EPI_RESLN_Q4, bias=p["b2"], residual=T["h1"], gamma=p["ln2_g"], beta=p["ln2_b"])
    assert_f16_close(T["h_out"], r3["f16"], "h_out")
    c, s, z = orc.quantize_rows_asym(T["h_out"])
    assert np.array_equal(T["hq_out"], c) and np.array_equal(T["hs_out"], s) and np.array_equal(T["hz_out"], z)


def test_asym_encoder_stack_host_device_graph(q4):
    """The asymmetric stack (W4A4Encoder(asym=True) -> q4_encoder_stack with asym_acts):
    device, host-buffer and graph replay agree bit for bit, and layer 0 equals q4_encoder_layer_asym."""
    cfg = dict(synth.BERT["base"])
    L, B, S = 2, 2, 128
    layers = [synth.layer_params(cfg, l, "astk") for l in range(L)]
    enc = q4.W4A4Encoder(cfg, layers, asym=True)
    x = synth.hidden(B * S, cfg["hidden"], "astk_x")
    xd = dev(x)
    out_d = torch.empty_like(xd)
    enc.forward(xd, out_d, B, S)
    xh = torch.from_numpy(x).pin_memory()
    out_h = torch.empty(xh.shape, dtype=torch.float16).pin_memory()
    enc.forward(xh, out_h, B, S)
    torch.cuda.synchronize()
    assert torch.equal(out_h, out_d.cpu())
    out_g = torch.empty_like(xd)
    enc.capture(xd, out_g, B, S)
    enc.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_g, out_d)
    # by hand: asym quantize + two asym layers
    xq, xs, xz = q4.quantize_rows_asym(xd)
    hcur = xd
    for l in range(L):
        o = q4.encoder_layer(enc.cfg, enc.weights[l], B, S, hcur, xq, xs, hz_in=xz)
        hcur, xq, xs, xz = o["h_out"], o["hq_out"], o["hs_out"], o["hz_out"]
    assert torch.equal(hcur, out_d)
