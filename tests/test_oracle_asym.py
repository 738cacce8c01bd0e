"""Pins for the asymmetric-activation oracle (O-15 / O-16):
hand-evaluated examples, exact-rational brute force, the invariants SPEC.md fixes (range
[0, 2^b - 1], roundtrip within scale/2, asym RMS <= sym RMS on all-positive data), Python-int
GEMMs and torch fp64 F.linear on the dequantized operands."""
from fractions import Fraction

import numpy as np
import torch
import torch.nn.functional as F

from paper_2301_12017_b200 import synth


def f16ulp_close(got, ref, ulps=1):
    a = np.asarray(got, np.float16).view(np.int16).astype(np.int64)
    b = np.asarray(ref, np.float16).view(np.int16).astype(np.int64)
    a = np.where(a < 0, -32768 - a, a)
    b = np.where(b < 0, -32768 - b, b)
    return np.abs(a - b).max() <= ulps


GOLD = [  # (x, codes, scale_num / 15, zero): PAPER.md:709-715 at b = 4 (R17, R18), by hand
    ([0.0, 1.0, 2.0, 3.0], [0, 5, 10, 15], 3.0, 0.0),      # SPEC.md:167 grid case at b = 4
    ([-1.0, 0.5, 2.0], [0, 8, 15], 3.0, -1.0),             # 5 (x + 1): 7.5 is a tie -> even 8
    ([5.0, 5.0, 5.0, 5.0], [0, 0, 0, 0], None, 5.0),       # constant row: scale 1
]


def test_asym_golden(orc):
    for x, codes, d, z in GOLD:
        c, s, zz = orc.quantize_rows_asym(np.array([x], np.float16))
        assert orc.unpack_u4(c, len(x))[0].tolist() == codes
        assert s[0] == (np.float32(1.0) if d is None else np.float32(d / 15.0))
        assert zz[0] == np.float32(z)


def test_asym_brute_force_and_invariants(orc):
    g = np.random.default_rng(21)
    for _ in range(60):
        x = np.array([g.standard_normal(37) * 10 ** g.uniform(-2, 2) + g.uniform(-3, 3)], np.float16)
        c, s, z = orc.quantize_rows_asym(x)
        q = orc.unpack_u4(c, 37)[0].astype(np.int64)
        xv = [Fraction(float(v)) for v in x[0]]
        mn, mx = min(xv), max(xv)
        assert q.tolist() == [round(15 * (v - mn) / (mx - mn)) for v in xv]
        assert q.min() == 0 and q.max() == 15 and z[0] == np.float32(float(mn))
        # |x - (min + D q / 15)| <= D / 30 exactly
        assert all(abs(v - (mn + (mx - mn) * int(qq) / 15)) <= (mx - mn) / 30 for v, qq in zip(xv, q))


def test_asym_rms_not_worse_on_positive_data(orc):
    """asymmetric <= symmetric RMS error on all-positive tensors."""
    g = np.random.default_rng(22)
    x = np.abs(g.standard_normal((64, 256))).astype(np.float16) + np.float16(0.5)
    c, s, z = orc.quantize_rows_asym(x)
    xa = z[:, None].astype(np.float64) + s[:, None].astype(np.float64) * orc.unpack_u4(c, 256)
    cs, ss = orc.quantize_rows(x)
    xs = ss[:, None].astype(np.float64) * orc.unpack_int4(cs, 256)
    xd = x.astype(np.float64)
    assert (np.sqrt(((xa - xd) ** 2).mean(1)) <= np.sqrt(((xs - xd) ** 2).mean(1)) + 1e-12).all()


def test_asym_linear_vs_ints_and_torch(orc):
    M, N, K = 40, 96, 256
    x = synth.hidden(M, K, "ta_x") + np.float16(1.0)
    wt = synth.weight(N, K, "ta_w")
    b = synth.bias(N, "ta_b")
    a, sa, za = orc.quantize_rows_asym(x)
    w, sw = orc.quantize_rows(wt)
    qa = orc.unpack_u4(a, K).astype(np.int64)
    qw = orc.unpack_int4(w, K).astype(np.int64)
    i32 = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_I32)["i32"]
    assert np.array_equal(i32, qa @ qw.T)
    ref_small = [[sum(int(qa[m, k]) * int(qw[n, k]) for k in range(K)) for n in range(3)] for m in range(3)]
    assert i32[:3, :3].tolist() == ref_small
    out = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_F16, bias=b)["f16"]
    dqa = torch.tensor(za, dtype=torch.float64)[:, None] + torch.tensor(sa, dtype=torch.float64)[:, None] * torch.tensor(qa, dtype=torch.float64)
    dqw = torch.tensor(sw, dtype=torch.float64)[:, None] * torch.tensor(qw, dtype=torch.float64)
    ref = F.linear(dqa, dqw, torch.tensor(b, dtype=torch.float64)).numpy()
    assert f16ulp_close(out, ref.astype(np.float16), 1)


def _asym_operands(orc, M, N, K, tag):
    x = synth.hidden(M, K, f"ae_x{tag}") + np.float16(0.25)
    a, sa, za = orc.quantize_rows_asym(x)
    w, sw = orc.quantize_rows(synth.weight(N, K, f"ae_w{tag}"))
    b = synth.bias(N, f"ae_b{tag}")
    # dequantized operands in fp64: za + sa qa (unsigned) and sw qw (signed)
    xd = za[:, None].astype(np.float64) + sa[:, None].astype(np.float64) * orc.unpack_u4(a, K)
    wd = sw[:, None].astype(np.float64) * orc.unpack_int4(w, K)
    t = torch.from_numpy(xd) @ torch.from_numpy(wd).T + torch.from_numpy(b.astype(np.float64))
    return a, sa, za, w, sw, b, t


def test_asym_gelu_requant_epilogue(orc):
    """O-16 GELU_Q4 (NEXT-3 asymmetric layer): fp16 = GELU(t) of the torch fp64 linear on the
    dequantized operands (<= 1 ulp), codes/scales/zeros = O-15 of that fp16 row (pinned above),
    and the symmetric-output variant codes the same fp16 with O-1."""
    M, N, K = 9, 96, 64
    a, sa, za, w, sw, b, t = _asym_operands(orc, M, N, K, "g")
    r = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_GELU_Q4, bias=b)
    ref = F.gelu(t).numpy().astype(np.float16)
    assert f16ulp_close(r["f16"], ref)
    c, s, z = orc.quantize_rows_asym(r["f16"])
    assert np.array_equal(r["codes"], c) and np.array_equal(r["scales"], s) and np.array_equal(r["zeros"], z)
    r2 = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_GELU_Q4, bias=b, asym_out=False)
    c2, s2 = orc.quantize_rows(r2["f16"])
    assert np.array_equal(r2["f16"], r["f16"]) and np.array_equal(r2["codes"], c2) and "zeros" not in r2


def test_asym_resln_requant_epilogue(orc):
    """O-16 RESLN_Q4: fp16 = LayerNorm(t + residual) (torch fp64, biased variance, eps 1e-12)."""
    M, N, K = 7, 128, 96
    a, sa, za, w, sw, b, t = _asym_operands(orc, M, N, K, "r")
    res = synth.hidden(M, N, "ae_res")
    g, bt = synth.ln_params(N, "ae_ln")
    r = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, orc.EPI_RESLN_Q4, bias=b, residual=res, gamma=g, beta=bt)
    z = t + torch.from_numpy(res.astype(np.float64))
    ref = F.layer_norm(z, (N,), torch.from_numpy(g.astype(np.float64)), torch.from_numpy(bt.astype(np.float64)),
                       eps=1e-12).numpy().astype(np.float16)
    assert f16ulp_close(r["f16"], ref)
    c, s, zz = orc.quantize_rows_asym(r["f16"])
    assert np.array_equal(r["codes"], c) and np.array_equal(r["scales"], s) and np.array_equal(r["zeros"], zz)


def test_asym_epilogues_reduce_to_symmetric(orc):
    """Zero points 0 and codes in [0, 7] are valid for both quantizers: the asymmetric linear
    then equals the symmetric oracle O-5..O-7 (pinned in test_oracle_gemm.py) element for element."""
    M, N, K = 6, 64, 64
    g = np.random.default_rng(23)
    q = g.integers(0, 8, (M, K)).astype(np.int8)
    a = orc.pack_int4(q)
    sa, za = (g.uniform(0.5, 2, M) / 7).astype(np.float32), np.zeros(M, np.float32)
    w, sw = orc.quantize_rows(synth.weight(N, K, "ae_sym_w"))
    b = synth.bias(N, "ae_sym_b")
    res = synth.hidden(M, N, "ae_sym_r")
    gm, bt = synth.ln_params(N, "ae_sym_ln")
    for epi, kw in ((orc.EPI_F16, {}), (orc.EPI_GELU_Q4, {}), (orc.EPI_RESLN_Q4, dict(residual=res, gamma=gm, beta=bt))):
        ra = orc.w4a4_asym_linear(a, sa, za, w, sw, M, N, K, epi, bias=b, asym_out=False, **kw)
        rs = orc.w4a4_linear(a, sa, w, sw, M, N, K, epi, bias=b, **kw)
        assert np.array_equal(ra["f16"], rs["f16"])
        if epi != orc.EPI_F16:
            assert np.array_equal(ra["codes"], rs["codes"]) and np.array_equal(ra["scales"], rs["scales"])
