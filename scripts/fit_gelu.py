"""Fit of the GELU tail polynomials in csrc/common.cuh (offline tooling; not part of the
product path).  GELU(x) = max(x,0) - |x| Q(|x|), Q(t) = exp(-t^2/2) R(t), R(v) a degree-DEG
polynomial in v = HI/2 - min(t, HI).  Weighted least squares on the GELU error, reweighted
towards minimax; prints the coefficients and the max |error| of the float32 evaluation order
the kernel uses against the fp64 erf form.

  python scripts/fit_gelu.py            # gelu16 (GELU_Q4 epilogue): HI 4.5, degree 6
  python scripts/fit_gelu.py 5.5 8 old  # gelu2 (row-per-thread epilogues)"""
import sys

import numpy as np
from scipy.special import erfc

HI = float(sys.argv[1]) if len(sys.argv) > 1 else 4.5
DEG = int(sys.argv[2]) if len(sys.argv) > 2 else 6
OLD = len(sys.argv) > 3  # gelu2: tn kept; gelu16: tn recovered as v - HI/2
t = np.linspace(0, HI, 200001)
R = 0.5 * erfc(t / np.sqrt(2)) * np.exp(t * t / 2)
V = np.vander(HI / 2 - t, DEG + 1)
w = t * np.exp(-t * t / 2) + 2e-3
c, *_ = np.linalg.lstsq(V * w[:, None], R * w, rcond=None)
for _ in range(30):
    e = np.abs((V @ c - R) * t * np.exp(-t * t / 2))
    w2 = w * (1 + 50 * e / e.max())
    c, *_ = np.linalg.lstsq(V * w2[:, None], R * w2, rcond=None)
c32 = c.astype(np.float32)
x = np.linspace(-8, 8, 400001).astype(np.float32)
tn = np.maximum(-np.abs(x), np.float32(-HI))
v = (tn + np.float32(HI / 2)).astype(np.float32)
r = np.full_like(v, c32[0])
for ci in c32[1:]:
    r = (r * v + ci).astype(np.float32)
if not OLD:
    tn = (v - np.float32(HI / 2)).astype(np.float32)
ea = ((tn * tn).astype(np.float32) * np.float32(-0.72134752044448170)).astype(np.float32)
q = (np.exp2(ea.astype(np.float64)).astype(np.float32) * r).astype(np.float32)
y = (tn * q + np.maximum(x, 0)).astype(np.float32)
xd = x.astype(np.float64)
print("coefficients (highest degree first):", ", ".join(f"{float(ci):.9e}f" for ci in c32))
print("max |GELU error| (float32 evaluation):", float(np.max(np.abs(y - xd * 0.5 * erfc(-xd / np.sqrt(2))))))
