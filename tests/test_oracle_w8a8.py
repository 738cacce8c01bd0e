"""Pins for the W8A8 oracle (O-11..O-13: the paper's INT8 baseline,
PAPER.md:406, 496-502) against things other than the oracle: hand-evaluated worked
examples (tests/golden/quantize_i8_examples.json, cited), brute force over the exact
rationals, invariants, Python-int GEMMs, the already-pinned 4-bit GEMM, and torch fp64
routines on the dequantized operands."""
import json
import os
from fractions import Fraction

import numpy as np
import torch
import torch.nn.functional as F

from paper_2301_12017_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "quantize_i8_examples.json")))


def f16ulp_close(got, ref, ulps=1):
    a = np.asarray(got, np.float16).view(np.int16).astype(np.int64)
    b = np.asarray(ref, np.float16).view(np.int16).astype(np.int64)
    a = np.where(a < 0, -32768 - a, a)
    b = np.where(b < 0, -32768 - b, b)
    return np.abs(a - b).max() <= ulps


def _rhe(fr: Fraction) -> int:
    """round half to even of an exact rational (Python's round does exactly this)."""
    return round(fr)


# ------------------------------------------------------------------ O-11
def test_quantize_i8_golden(orc):
    for ex in GOLD["quantize"]:
        x = np.array([ex["x"]], np.float16)
        c, s = orc.quantize_rows_i8(x)
        assert c[0].tolist() == ex["codes"], ex["cite"]
        assert s[0] == np.float32(ex["scale_num"]) / np.float32(ex["scale_den"]), ex["cite"]


def test_quantize_i8_brute_force_exact_rationals(orc):
    g = np.random.default_rng(11)
    rows = [g.standard_normal(33) * 10 ** g.uniform(-3, 3) for _ in range(40)]
    # rows built on exact ties of 127 x / amax: amax = 127 * 2^-4 (fp16-exact), x = (k + 1/2) 2^-4
    rows.append(np.concatenate([[127 / 16], (np.arange(-20, 20) + 0.5) / 16]))
    for clip in (0.0, 1.5):
        for r in rows:
            x = np.array([r], np.float16)
            c, s = orc.quantize_rows_i8(x, clip=clip)
            xv = [Fraction(float(v)) for v in x[0]]
            if clip:
                xv = [max(min(v, Fraction(clip)), Fraction(-clip)) for v in xv]
            a = max(abs(v) for v in xv)
            ref = [0] * len(xv) if a == 0 else [_rhe(127 * v / a) for v in xv]
            assert c[0].tolist() == ref
            assert s[0] == (np.float32(1.0) if a == 0 else np.float32(float(a)) / np.float32(127))


def test_quantize_i8_invariants_and_idempotence(orc):
    x = synth.hidden(256, 1024, "t_i8_inv")
    c, s = orc.quantize_rows_i8(x)
    assert c.min() >= -127 and c.max() <= 127
    assert (np.abs(c).max(1) == 127).all()  # the amax element maps to +-127
    xd = x.astype(np.float64)
    amax = np.abs(xd).max(1, keepdims=True)
    # |x - (a/127) q| <= a/254 exactly; with the stored fp32 scale s = fl32(a/127) the
    # product s q (|q| <= 127) moves by at most 127 * 2^-24 s, hence the 2^-16 slack
    assert (np.abs(xd - amax / 127 * c) <= amax / 254 * (1 + 1e-12)).all()
    err = np.abs(xd - s.astype(np.float64)[:, None] * c)
    assert (err <= s.astype(np.float64)[:, None] / 2 * (1 + 2 ** -16)).all()
    o = np.argsort(xd[0])  # monotone within a row
    assert (np.diff(c[0][o].astype(np.int64)) >= 0).all()
    # idempotent on already-quantized data (fp16 grid, amax >= 2^-14)
    y = (s[:, None].astype(np.float64) * c).astype(np.float16)
    c2, s2 = orc.quantize_rows_i8(y)
    assert np.array_equal(c2, c)


# ------------------------------------------------------------------ O-12
def test_gemm_i8_python_ints_and_extremes(orc):
    g = np.random.default_rng(12)
    for (M, N, K) in ((3, 5, 7), (4, 9, 32), (1, 1, 1)):
        a = g.integers(-127, 128, (M, K), dtype=np.int8)
        w = g.integers(-127, 128, (N, K), dtype=np.int8)
        acc = orc.gemm_i32_i8(a, w, M, N, K)
        ref = [[sum(int(a[m, k]) * int(w[n, k]) for k in range(K)) for n in range(N)] for m in range(M)]
        assert acc.tolist() == ref
    K = 4096  # all -128: 2^14 * K = 2^26 < 2^31
    a = np.full((2, K), -128, np.int8)
    assert (orc.gemm_i32_i8(a, a, 2, 2, K) == 16384 * K).all()


def test_gemm_i8_agrees_with_pinned_int4_gemm(orc):
    """On codes inside the 4-bit range the 8-bit GEMM equals the (independently pinned)
    packed INT4 GEMM."""
    g = np.random.default_rng(13)
    M, N, K = 17, 40, 256
    qa = g.integers(-8, 8, (M, K), dtype=np.int8)
    qw = g.integers(-8, 8, (N, K), dtype=np.int8)
    acc4 = orc.gemm_i32(orc.pack_int4(qa), orc.pack_int4(qw), M, N, K)
    assert np.array_equal(orc.gemm_i32_i8(qa, qw, M, N, K), acc4)


# ------------------------------------------------------------------ O-13
def _dq(codes, scales):
    return torch.tensor(codes, dtype=torch.float64) * torch.tensor(scales, dtype=torch.float64)[:, None]


def test_w8a8_f16_fake_quant_parity(orc):
    M, N, K = 64, 96, 768
    x, wt, b = synth.hidden(M, K, "t8_fq"), synth.weight(N, K, "t8_fq_w"), synth.bias(N, "t8_fq_b")
    a, sa = orc.quantize_rows_i8(x)
    w, sw = orc.quantize_rows_i8(wt)
    out = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_F16, bias=b)
    ref = F.linear(_dq(a, sa), _dq(w, sw), torch.tensor(b, dtype=torch.float64)).numpy()
    assert f16ulp_close(out["f16"], ref.astype(np.float16), 1)
    i32 = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_I32)["i32"]
    assert np.array_equal(i32, a.astype(np.int64) @ w.astype(np.int64).T)


def test_w8a8_gelu_and_resln_epilogues(orc):
    g = np.random.default_rng(14)
    M, N, K = 40, 512, 256
    a = g.integers(-127, 128, (M, K), dtype=np.int8)
    w = g.integers(-127, 128, (N, K), dtype=np.int8)
    sa = synth.random_scales(M, "t8_sa") / 16
    sw = synth.random_scales(N, "t8_sw") / 16
    b = synth.bias(N, "t8_b")
    acc = (a.astype(np.float64) @ w.astype(np.float64).T)
    t = torch.tensor(acc * sa.astype(np.float64)[:, None] * sw.astype(np.float64)[None, :] + b.astype(np.float64))
    out = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_GELU_Q4, bias=b)
    assert f16ulp_close(out["f16"], F.gelu(t, approximate="none").numpy().astype(np.float16), 1)
    assert np.abs(t.numpy()).max() > 3
    c2, s2 = orc.quantize_rows_i8(out["f16"])  # R13 at 8 bits
    assert np.array_equal(c2, out["codes"]) and np.array_equal(s2, out["scales"])
    res = synth.hidden(M, N, "t8_res")
    gam, bet = synth.ln_params(N, "t8_ln")
    out = orc.w8a8_linear(a, sa, w, sw, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res, gamma=gam, beta=bet)
    z = t + torch.tensor(res.astype(np.float64))
    ref = F.layer_norm(z, (N,), torch.tensor(gam, dtype=torch.float64), torch.tensor(bet, dtype=torch.float64), eps=1e-12)
    assert f16ulp_close(out["f16"], ref.numpy().astype(np.float16), 1)
    c2, s2 = orc.quantize_rows_i8(out["f16"])
    assert np.array_equal(c2, out["codes"]) and np.array_equal(s2, out["scales"])


# ------------------------------------------------------------------ O-14 (FP16 parts, NEXT-1)
def test_f16_linear_vs_torch_fp64(orc):
    """The unquantized linear of a per-part strategy: fp64 F.linear on the fp16 operands
    (1 fp16 ulp), torch F.gelu / F.layer_norm for the fused epilogues, codes = O-1(y)."""
    M, N, K = 48, 512, 384
    a, w = synth.hidden(M, K, "t16_a"), synth.weight(N, K, "t16_w") * 8
    b = synth.bias(N, "t16_b")
    t = F.linear(torch.tensor(a, dtype=torch.float64), torch.tensor(w, dtype=torch.float64),
                 torch.tensor(b, dtype=torch.float64))
    out = orc.f16_linear(a, w, M, N, K, orc.EPI_F16, bias=b)
    assert f16ulp_close(out["f16"], t.numpy().astype(np.float16), 1)
    out = orc.f16_linear(a, w, M, N, K, orc.EPI_GELU_Q4, bias=b)
    assert f16ulp_close(out["f16"], F.gelu(t, approximate="none").numpy().astype(np.float16), 1)
    c2, s2 = orc.quantize_rows(out["f16"])
    assert np.array_equal(c2, out["codes"]) and np.array_equal(s2, out["scales"])
    res = synth.hidden(M, N, "t16_r")
    gam, bet = synth.ln_params(N, "t16_ln")
    out = orc.f16_linear(a, w, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res, gamma=gam, beta=bet)
    ref = F.layer_norm(t + torch.tensor(res.astype(np.float64)), (N,), torch.tensor(gam, dtype=torch.float64),
                       torch.tensor(bet, dtype=torch.float64), eps=1e-12)
    assert f16ulp_close(out["f16"], ref.numpy().astype(np.float16), 1)
    c2, s2 = orc.quantize_rows(out["f16"])
    assert np.array_equal(c2, out["codes"]) and np.array_equal(s2, out["scales"])
    # an fp16 operand pair that is exactly an INT4 problem gives the W4A4 oracle's result
    g = np.random.default_rng(15)
    qa = g.integers(-7, 8, (M, K)).astype(np.int8)
    qw = g.integers(-7, 8, (N, K)).astype(np.int8)
    f = orc.f16_linear(qa.astype(np.float16), qw.astype(np.float16), M, N, K, orc.EPI_F16)["f16"]
    q = orc.w4a4_linear(orc.pack_int4(qa), np.ones(M, np.float32), orc.pack_int4(qw), np.ones(N, np.float32),
                        M, N, K, orc.EPI_F16)["f16"]
    assert np.array_equal(f, q)
