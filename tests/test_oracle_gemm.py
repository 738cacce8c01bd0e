"""Pins for oracle O-4 (integer GEMM), O-5..O-7 (fused epilogues), O-8 (attention)
and O-9 (encoder layer) against brute force, closed forms, special cases from the
spec and torch float64 library routines (F.linear, F.gelu,
F.layer_norm, F.scaled_dot_product_attention) applied to the dequantized operands."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2301_12017_b200 import synth


def f16ulp_close(got, ref, ulps=1):
    """fp16 arrays equal up to `ulps` units in the last place (ordered-int distance)."""
    a = got.astype(np.float16).view(np.int16).astype(np.int32)
    b = ref.astype(np.float16).view(np.int16).astype(np.int32)
    a = np.where(a < 0, -32768 - a, a)
    b = np.where(b < 0, -32768 - b, b)
    return np.abs(a - b).max() <= ulps


def _rand_codes(g, rows, cols):
    return g.integers(0, 256, size=(rows, cols // 2), dtype=np.uint8)


# ------------------------------------------------------------------ O-4
def test_gemm_identity_and_ones(orc):
    K = 16
    eye = np.eye(K, dtype=np.int8)
    g = np.random.default_rng(0)
    m = g.integers(-8, 8, (5, K)).astype(np.int8)
    acc = orc.gemm_i32(orc.pack_int4(m), orc.pack_int4(eye), 5, K, K)
    assert np.array_equal(acc, m.astype(np.int32))  # identity x m -> m
    ones = np.ones((2, 2), np.int8)
    acc = orc.gemm_i32(orc.pack_int4(ones), orc.pack_int4(ones), 2, 2, 2)
    assert (acc == 2).all()


def test_gemm_brute_force_python_ints(orc):
    g = np.random.default_rng(1)
    for _ in range(40):  # random shapes <= 64 vs a triple loop
        M, N = int(g.integers(1, 65)), int(g.integers(1, 65))
        K = 2 * int(g.integers(1, 33))
        a = g.integers(-8, 8, (M, K))
        w = g.integers(-8, 8, (N, K))
        acc = orc.gemm_i32(orc.pack_int4(a.astype(np.int8)), orc.pack_int4(w.astype(np.int8)), M, N, K)
        ref = [[sum(int(a[i, k]) * int(w[j, k]) for k in range(K)) for j in range(N)] for i in range(M)]
        assert acc.tolist() == ref


def test_gemm_extremes_and_numpy(orc):
    K = 4096
    m8 = np.full((3, K // 2), 0x88, np.uint8)  # all -8
    acc = orc.gemm_i32(m8, m8, 3, 3, K)
    assert (acc == 64 * K).all()  # |acc| bound 64K (SURVEY O-4)
    g = np.random.default_rng(2)
    a, w = _rand_codes(g, 64, 1024), _rand_codes(g, 96, 1024)
    acc = orc.gemm_i32(a, w, 64, 96, 1024)
    qa = orc.unpack_int4(a, 1024).astype(np.int64)
    qw = orc.unpack_int4(w, 1024).astype(np.int64)
    assert np.array_equal(acc, (qa @ qw.T).astype(np.int32))


# ------------------------------------------------------------------ O-5
def test_f16_epilogue_unit_scales_is_float_acc(orc):
    g = np.random.default_rng(3)
    M, N, K = 8, 16, 32
    a, w = _rand_codes(g, M, K), _rand_codes(g, N, K)
    out = orc.w4a4_linear(a, np.ones(M, np.float32), w, np.ones(N, np.float32), M, N, K,
                          orc.EPI_F16)
    acc = orc.gemm_i32(a, w, M, N, K)  # |acc| <= 64*32 = 2048: exact in fp16
    assert np.array_equal(out["f16"].astype(np.float64), acc.astype(np.float64))


def test_f16_epilogue_fake_quant_parity(orc):
    """float64 F.linear(dequant(qa), dequant(qw), b) vs the fused oracle."""
    g = np.random.default_rng(4)
    M, N, K = 64, 96, 768
    x = synth.hidden(M, K, "t_fq")
    wt = synth.weight(N, K, "t_fq_w")
    b = synth.bias(N, "t_fq_b")
    a, sa = orc.quantize_rows(x)
    w, sw = orc.quantize_rows(wt)
    out = orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_F16, bias=b)
    dqa = torch.tensor(orc.unpack_int4(a, K), dtype=torch.float64) * torch.tensor(sa, dtype=torch.float64)[:, None]
    dqw = torch.tensor(orc.unpack_int4(w, K), dtype=torch.float64) * torch.tensor(sw, dtype=torch.float64)[:, None]
    ref = F.linear(dqa, dqw, torch.tensor(b, dtype=torch.float64)).numpy()
    assert f16ulp_close(out["f16"], ref.astype(np.float16), 1)


# ------------------------------------------------------------------ O-6
def test_gelu_q4_epilogue(orc):
    g = np.random.default_rng(5)
    M, N, K = 48, 256, 256
    a, w = _rand_codes(g, M, K), _rand_codes(g, N, K)
    sa = synth.random_scales(M, "t_g_sa") * 4
    sw = synth.random_scales(N, "t_g_sw")
    b = synth.bias(N, "t_g_b")
    out = orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_GELU_Q4, bias=b)
    acc = orc.gemm_i32(a, w, M, N, K).astype(np.float64)
    t = torch.tensor(acc * sa.astype(np.float64)[:, None] * sw.astype(np.float64)[None, :] + b.astype(np.float64))
    ref = F.gelu(t, approximate="none").numpy()  # erf GELU (reading R11)
    assert f16ulp_close(out["f16"], ref.astype(np.float16), 1)
    assert np.abs(t.numpy()).max() > 3  # exercises the tails
    # codes/scales are O-1 applied to the stored fp16 GELU output (reading R13)
    c2, s2 = orc.quantize_rows(out["f16"])
    assert np.array_equal(c2, out["codes"]) and np.array_equal(s2, out["scales"])
    # closed forms: gelu(0) = 0, gelu(x) -> x for large x
    z = orc.w4a4_linear(np.zeros((1, K // 2), np.uint8), np.ones(1, np.float32), w[:1],
                        np.ones(1, np.float32), 1, 1, K, orc.EPI_GELU_Q4,
                        bias=np.array([8.0], np.float16))
    assert z["f16"][0, 0] == np.float16(8.0)
    z0 = orc.w4a4_linear(np.zeros((1, K // 2), np.uint8), np.ones(1, np.float32), w[:1],
                         np.ones(1, np.float32), 1, 1, K, orc.EPI_GELU_Q4)
    assert z0["f16"][0, 0] == 0 and z0["scales"][0] == 1.0


# ------------------------------------------------------------------ O-7
def test_resln_q4_epilogue(orc):
    g = np.random.default_rng(6)
    M, N, K = 40, 768, 256
    a, w = _rand_codes(g, M, K), _rand_codes(g, N, K)
    sa = synth.random_scales(M, "t_l_sa")
    sw = synth.random_scales(N, "t_l_sw")
    b = synth.bias(N, "t_l_b")
    res = synth.hidden(M, N, "t_l_res")
    gam, bet = synth.ln_params(N, "t_l_ln")
    out = orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res,
                          gamma=gam, beta=bet, ln_eps=1e-12)
    acc = orc.gemm_i32(a, w, M, N, K).astype(np.float64)
    z = torch.tensor(acc * sa.astype(np.float64)[:, None] * sw.astype(np.float64) + b.astype(np.float64) + res.astype(np.float64))
    ref = F.layer_norm(z, (N,), torch.tensor(gam, dtype=torch.float64), torch.tensor(bet, dtype=torch.float64), eps=1e-12).numpy()
    assert f16ulp_close(out["f16"], ref.astype(np.float16), 1)
    c2, s2 = orc.quantize_rows(out["f16"])
    assert np.array_equal(c2, out["codes"]) and np.array_equal(s2, out["scales"])
    # pre-affine moments: mean 0 and var 1
    one = np.ones(N, np.float16)
    zer = np.zeros(N, np.float16)
    o2 = orc.w4a4_linear(a, sa, w, sw, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res,
                         gamma=one, beta=zer)
    y = o2["f16"].astype(np.float64)
    assert np.abs(y.mean(1)).max() < 1e-3 and np.abs(y.var(1) - 1).max() < 5e-4
    # constant row -> beta: zero codes, zero bias, constant residual
    cres = np.full((1, N), 3.25, np.float16)
    o3 = orc.w4a4_linear(np.zeros((1, K // 2), np.uint8), np.ones(1, np.float32), w, sw, 1, N, K,
                         orc.EPI_RESLN_Q4, residual=cres, gamma=gam, beta=bet)
    assert np.array_equal(o3["f16"][0], bet)
    # gamma = 0 -> beta
    o4 = orc.w4a4_linear(a[:2], sa[:2], w, sw, 2, N, K, orc.EPI_RESLN_Q4, bias=b,
                         residual=res[:2], gamma=zer, beta=bet)
    assert np.array_equal(o4["f16"], np.stack([bet, bet]))
    # [1,2,3,4] normalises to (x - 2.5)/sqrt(1.25)
    o5 = orc.w4a4_linear(np.zeros((1, 16), np.uint8), np.ones(1, np.float32),
                         np.zeros((4, 16), np.uint8), np.ones(4, np.float32), 1, 4, 32,
                         orc.EPI_RESLN_Q4, residual=np.array([[1, 2, 3, 4]], np.float16),
                         gamma=np.ones(4, np.float16), beta=np.zeros(4, np.float16))
    want = ((np.arange(1, 5) - 2.5) / np.sqrt(1.25 + 1e-12)).astype(np.float16)
    assert np.array_equal(o5["f16"][0], want)


# ------------------------------------------------------------------ O-8
def _sdpa_ref(qkv, B, S, H, d):
    t = torch.tensor(qkv.astype(np.float64)).view(B, S, 3, H, d)
    q, k, v = (t[:, :, i].transpose(1, 2) for i in range(3))
    o = F.scaled_dot_product_attention(q, k, v)  # softmax(QK^T/sqrt(d)) V, no mask
    return o.transpose(1, 2).reshape(B * S, H * d).numpy()


def test_attention_vs_sdpa(orc):
    B, S, H, d = 2, 128, 4, 64
    qkv = synth.hidden(B * S, 3 * H * d, "t_att")
    ctx, codes, scales = orc.attention(qkv, B, S, H, d)
    ref = _sdpa_ref(qkv, B, S, H, d)
    assert f16ulp_close(ctx, ref.astype(np.float16), 1)
    c2, s2 = orc.quantize_rows(ctx)  # per-token quantize over all heads
    assert np.array_equal(c2, codes) and np.array_equal(s2, scales)


def test_attention_special_cases(orc):
    H, d = 2, 64
    # T = 1 -> probability 1, ctx = V
    qkv = synth.hidden(3, 3 * H * d, "t_att1")
    ctx, _, _ = orc.attention(qkv, 3, 1, H, d)
    assert np.array_equal(ctx, qkv[:, 2 * H * d:])
    # uniform scores (q = 0) -> ctx = mean of V
    S = 16
    qkv = synth.hidden(S, 3 * H * d, "t_att2")
    qkv[:, : H * d] = 0
    ctx, _, _ = orc.attention(qkv, 1, S, H, d)
    mean_v = qkv[:, 2 * H * d:].astype(np.float64).mean(0)
    assert f16ulp_close(ctx, np.broadcast_to(mean_v, ctx.shape).astype(np.float16), 1)


# ------------------------------------------------------------------ O-9
def test_encoder_layer_teacher_forced_vs_torch(orc):
    """Each stage of the oracle layer equals the torch float64 op on that stage's
    (oracle-produced) inputs: F.linear / sdpa / layer_norm / gelu on dequantized codes."""
    cfg = dict(synth.BERT["base"])
    cfg.update(hidden=256, heads=4, ffn=1024)
    B, S = 2, 64
    M, h, f = B * S, cfg["hidden"], cfg["ffn"]
    p = synth.layer_params(cfg, 0, "t_enc")
    w = dict(p)
    for k in ("wqkv", "wo", "w1", "w2"):
        w[k], w["s" + k[1:]] = orc.quantize_rows(p[k])
    x = synth.hidden(M, h, "t_enc_x")
    xq, xs = orc.quantize_rows(x)
    out = orc.encoder_layer(cfg, w, B, S, x, xq, xs, taps=True)
    D = lambda c, s, n: torch.tensor(orc.unpack_int4(c, n), dtype=torch.float64) * torch.tensor(s, dtype=torch.float64)[:, None]
    T = lambda a: torch.tensor(a.astype(np.float64))
    qkv = F.linear(D(xq, xs, h), D(w["wqkv"], w["sqkv"], h), T(p["bqkv"])).numpy()
    assert f16ulp_close(out["qkv"], qkv.astype(np.float16))
    ctx = _sdpa_ref(out["qkv"], B, S, cfg["heads"], cfg["head_dim"])
    assert f16ulp_close(out["ctx"], ctx.astype(np.float16))
    z = F.linear(D(out["ctx_codes"], out["ctx_scales"], h), D(w["wo"], w["so"], h), T(p["bo"])) + T(x)
    h1 = F.layer_norm(z, (h,), T(p["ln1_g"]), T(p["ln1_b"]), eps=1e-12).numpy()
    assert f16ulp_close(out["h1"], h1.astype(np.float16))
    f1 = F.gelu(F.linear(D(out["h1_codes"], out["h1_scales"], h), D(w["w1"], w["s1"], h), T(p["b1"]))).numpy()
    assert f16ulp_close(out["ffn1"], f1.astype(np.float16))
    z2 = F.linear(D(out["f_codes"], out["f_scales"], f), D(w["w2"], w["s2"], f), T(p["b2"])) + T(out["h1"])
    ho = F.layer_norm(z2, (h,), T(p["ln2_g"]), T(p["ln2_b"]), eps=1e-12).numpy()
    assert f16ulp_close(out["h_out"], ho.astype(np.float16))
    for tap, c, s in (("ctx", "ctx_codes", "ctx_scales"), ("h1", "h1_codes", "h1_scales"),
                      ("ffn1", "f_codes", "f_scales"), ("h_out", "hq_out", "hs_out")):
        c2, s2 = orc.quantize_rows(out[tap])
        assert np.array_equal(c2, out[c]) and np.array_equal(s2, out[s]), tap
