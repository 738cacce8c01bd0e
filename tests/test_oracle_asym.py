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
