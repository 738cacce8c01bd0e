"""Pins for oracle O-1 (quantize) and O-2 (pack) against things other than the oracle:
worked examples from the paper's spec (tests/golden, cited), brute force over the
integer grid, the IEEE fp32-division realisation over every fp16 pair, numpy's fp16
conversion, and the invariants the north_star fixes (codes in [-8,7],
|x - dequant(quant(x))| <= scale/2, idempotence)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "quantize_examples.json")))


def _codes(orc, packed, cols):
    return orc.unpack_int4(packed, cols).astype(np.int64)


# ------------------------------------------------------------------ fp16 conversion
def test_f16_to_f64_all_bit_patterns(orc):
    bits = np.arange(65536, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([orc.f16_to_f64(int(b)) for b in bits])
    finite = np.isfinite(ref)
    assert np.array_equal(got[finite], ref[finite])
    assert np.array_equal(np.isinf(got), np.isinf(ref))
    assert np.array_equal(np.isnan(got), np.isnan(ref))


def test_f64_to_f16_matches_numpy_rne(orc):
    # every finite positive fp16, the midpoints between neighbours (ties -> even),
    # values just off the midpoints, subnormals, and overflow
    pos = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = (pos[:-1] + pos[1:]) / 2
    extra = np.array([65504.0, 65519.99, 65520.0, 65536.0, 1e6, 2.0 ** -25, 2.0 ** -26,
                      3 * 2.0 ** -26, 1e-9, 0.0])
    vals = np.concatenate([pos, mids, np.nextafter(mids, 0), np.nextafter(mids, 1e9), extra])
    vals = np.concatenate([vals, -vals])
    ref = vals.astype(np.float16).view(np.uint16)
    got = np.array([orc.f64_to_f16_bits(v) for v in vals], np.uint16)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (vals[bad[:5]], got[bad[:5]], ref[bad[:5]])


# ------------------------------------------------------------------ golden examples
@pytest.mark.parametrize("ex", GOLD["quantize"], ids=lambda e: e["cite"][:40])
def test_quantize_golden(orc, ex):
    x = np.array([ex["x"]], np.float16)
    codes, scales = orc.quantize_rows(x)
    assert list(_codes(orc, codes, x.shape[1])[0]) == ex["codes"], ex["cite"]
    want = np.float32(ex["scale_num"]) / np.float32(ex["scale_den"])
    assert scales[0] == want, ex["cite"]


@pytest.mark.parametrize("ex", GOLD["pack"], ids=lambda e: e["cite"][:30])
def test_pack_golden(orc, ex):
    q = np.array([ex["q"]], np.int8)
    p = orc.pack_int4(q)
    assert list(p[0]) == ex["bytes"], ex["cite"]
    assert list(orc.unpack_int4(p, q.shape[1])[0]) == ex["q"]


def test_pack_exhaustive_byte_roundtrip(orc):
    # every byte value is a valid pair of nibbles; unpack -> pack is the identity
    allb = np.arange(256, dtype=np.uint8).reshape(1, 256)
    q = orc.unpack_int4(allb, 512)
    assert q.min() == -8 and q.max() == 7
    assert np.array_equal(orc.pack_int4(q), allb)
    # and nibble semantics: two's complement, low nibble = even index
    lo = np.array([((b & 15) ^ 8) - 8 for b in range(256)])
    hi = np.array([((b >> 4) ^ 8) - 8 for b in range(256)])
    assert np.array_equal(q[0, 0::2], lo) and np.array_equal(q[0, 1::2], hi)


def test_pack_out_of_range_names_coordinates(orc):
    q = np.zeros((3, 5), np.int8)
    q[2, 3] = 9
    with pytest.raises(ValueError, match=r"\(2, 3\)"):
        orc.pack_int4(q)


# ------------------------------------------------------------------ brute force
def _brute_code(x: Fraction, amax: Fraction) -> int:
    """Nearest point of the grid {k * amax/7 : k in [-8, 7]}, ties to the even k."""
    best = None
    for k in range(-8, 8):
        d = abs(x - Fraction(k) * amax / 7)
        if best is None or d < best[0] or (d == best[0] and k % 2 == 0):
            best = (d, k)
    return best[1]


def test_quantize_brute_force_small(orc):
    g = np.random.default_rng(7)
    rows = []
    for r in range(300):
        n = int(g.integers(1, 12))
        x = (g.standard_normal(n) * np.exp(g.normal(0, 2))).astype(np.float16)
        if r % 10 == 0:  # plant exact ties at k + 1/2 grid points
            a = np.float16(7.0 * 2.0 ** int(g.integers(-6, 6)))
            x = np.concatenate([[a], (np.float16(a / 7) * (g.integers(-13, 14, n) / 2)).astype(np.float16)])
            x = np.clip(x, -a, a).astype(np.float16)
        rows.append(x)
    for x in rows:
        codes, scales = orc.quantize_rows(x[None, :])
        got = _codes(orc, codes, x.size)[0]
        fx = [Fraction(float(v)) for v in x]
        amax = max(abs(v) for v in fx)
        if amax == 0:
            assert (got == 0).all() and scales[0] == 1.0
            continue
        want = [_brute_code(v, amax) for v in fx]
        assert list(got) == want, (x, got, want)
        assert scales[0] == np.float32(float(amax)) / np.float32(7.0)


# ------------------------------------------------------------------ exhaustive fp16
@pytest.mark.slow
def test_quantize_exhaustive_equals_fp32_division(orc):
    """Every (x, amax) fp16 pair with 0 <= x <= amax: the oracle's exact rational
    rounding equals rint(fl32(fl32(7x) / amax)) -- IEEE division, an independent
    realisation (SURVEY F3 found 0 mismatches; 105,182 exact ties make the tie rule
    matter).  Rows are [amax, all x <= amax] so the row's amax is the pair's amax."""
    allpos = np.arange(1, 0x7C00, dtype=np.uint16).view(np.float16)  # positive finite
    n = allpos.size
    chunk = 256
    ties = 0
    for s in range(0, n, chunk):
        idx = np.arange(s, min(n, s + chunk))
        width = idx[-1] + 1
        X = np.zeros((idx.size, width), np.float16)
        for r, i in enumerate(idx):
            X[r, : i + 1] = allpos[: i + 1]
        codes, scales = orc.quantize_rows(X, threads=0)
        q = orc.unpack_int4(codes, width).astype(np.int64)
        a = allpos[idx].astype(np.float32)[:, None]
        t = np.float32(7.0) * X.astype(np.float32)
        ref = np.rint(t / a)
        mask = np.arange(width)[None, :] <= idx[:, None]
        assert np.array_equal(q[mask], ref[mask].astype(np.int64)), f"chunk {s}"
        assert np.array_equal(scales, allpos[idx].astype(np.float32) / np.float32(7))
        # negated rows give the negated codes (symmetric mapping)
        if s % (chunk * 16) == 0:
            codes_n, _ = orc.quantize_rows(-X)
            qn = orc.unpack_int4(codes_n, width).astype(np.int64)
            assert np.array_equal(qn[mask], -q[mask])
        # count exact ties 7x/a = k + 1/2, via integers (fp16 = int * 2^-24)
        Xi = (X.astype(np.float64) * 2.0 ** 24).astype(np.int64)
        Ai = (allpos[idx].astype(np.float64) * 2.0 ** 24).astype(np.int64)[:, None]
        ties += int(((2 * 7 * Xi) % (2 * Ai) == Ai)[mask].sum())
    # SURVEY A.5 counts 105,182 ties over +-x; the sweep above covers x >= 0 only
    assert 2 * ties == 105182


# ------------------------------------------------------------------ invariants
def _rand_rows(seed, rows=2000, cols=64):
    g = np.random.default_rng(seed)
    x = g.standard_normal((rows, cols)) * np.exp(g.normal(0, 3, (rows, 1)))
    x[::17, :] = 0.0
    x[::23, 5] *= 40.0
    return np.clip(x, -60000, 60000).astype(np.float16)


def test_quantize_invariants(orc):
    x = _rand_rows(1)  # 2000 rows x 64 = 128k elements
    codes, scales = orc.quantize_rows(x)
    q = _codes(orc, codes, x.shape[1])
    assert q.min() >= -8 and q.max() <= 7  # range containment (north_star: codes clamp to [-8,7])
    xi = (np.abs(x.astype(np.float64)) * 2.0 ** 24).astype(np.int64) * np.sign(x.astype(np.float64)).astype(np.int64)
    A = np.abs(xi).max(axis=1, keepdims=True)
    nz = A[:, 0] > 0
    # |x - (amax/7) q| <= amax/14 exactly  <=>  2|7X - A q| <= A
    assert (2 * np.abs(7 * xi[nz] - A[nz] * q[nz]) <= A[nz]).all()
    # with the stored fp32 scale: |x - s q| <= (s/2)(1 + 2^-20)  (north_star: <= scale/2)
    s = scales.astype(np.float64)[:, None]
    err = np.abs(x.astype(np.float64) - s * q)
    assert (err[nz] <= s[nz] / 2 * (1 + 2.0 ** -20)).all()
    # monotone within a row
    order = np.argsort(x.astype(np.float64), axis=1, kind="stable")
    qs = np.take_along_axis(q, order, axis=1)
    assert (np.diff(qs, axis=1) >= 0).all()
    # zero rows -> scale 1, codes 0
    assert (scales[~nz] == 1.0).all() and (q[~nz] == 0).all()


def test_quantize_idempotent(orc):
    """quantize(fp16(scale * q)) returns the same codes and scale (north_star), for
    amax >= 2^-14 (below that fp16 cannot hold scale*q)."""
    x = _rand_rows(2)
    codes, scales = orc.quantize_rows(x)
    q = _codes(orc, codes, x.shape[1])
    amax = np.abs(x.astype(np.float32)).max(axis=1)
    keep = amax >= 2.0 ** -14
    deq = (scales[:, None].astype(np.float64) * q).astype(np.float16)
    codes2, scales2 = orc.quantize_rows(deq[keep])
    assert np.array_equal(_codes(orc, codes2, x.shape[1]), q[keep])
    assert np.array_equal(scales2, scales[keep])


def test_clip(orc):
    x = np.array([[10.0, -6.0, 2.5, -1.0]], np.float16)
    codes, scales = orc.quantize_rows(x, clip=5.0)  # PAPER.md:547 clip [-5, 5]
    assert list(_codes(orc, codes, 4)[0]) == [7, -7, 4, -1]  # 7*2.5/5=3.5 -> 4 (even)
    assert scales[0] == np.float32(5.0) / np.float32(7.0)
    with pytest.raises(ValueError):
        orc.quantize_rows(x, clip=0.1)  # 0.1 is not fp16-representable
