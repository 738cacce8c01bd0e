"""Attention trace at small batch (one head per CTA): per-CTA phase times of head 0 (Q4_TRACE
dump of scripts/probe_attn.py B S H, profiling build)."""
import sys, numpy as np
raw = np.frombuffer(open(sys.argv[1], "rb").read(), np.uint64).astype(np.float64)
rec = 512 * 16 * 16
n = int(sys.argv[2])
t = raw[-rec:].reshape(512, 16, 16)[:n]
h = t[:, 0, :]
t0 = h[:, 6].min()
rel = lambda k: (h[:, k] - t0) / 1e3
print("CTA entry (softmax warps)  min %.2f max %.2f us" % (rel(6).min(), rel(6).max()))
for nm, a, b in (("entry -> wait S start", 6, 0), ("wait S (TMA + QK^T)", 0, 1), ("softmax", 1, 2),
                 ("-> epilogue start", 2, 3), ("wait O (PV)", 3, 4), ("O tmem ld", 4, 8), ("normalize+pack", 8, 9),
                 ("store", 9, 5)):
    d = (h[:, b] - h[:, a]) / 1e3
    print(f"{nm:26s} mean {d.mean():.2f} us  (min {d.min():.2f} max {d.max():.2f})")
print("head done (from first entry): max %.2f us" % rel(5).max())
k = t[:, 15, :]
kt0 = k[:, 0].min()
kr = lambda i: (k[:, i] - kt0) / 1e3
print("kernel entry: min %.2f max %.2f us (first CTA = 0)" % (kr(0).min(), kr(0).max()))
for nm, a, b in (("prologue (barriers, TMEM alloc)", 0, 1), ("-> tail cluster barrier 1", 1, 2),
                 ("row scales (DSMEM reads)", 2, 3), ("codes", 3, 4), ("cluster barrier 2 + exit", 4, 5)):
    d = (k[:, b] - k[:, a]) / 1e3
    print(f"{nm:34s} mean {d.mean():.2f} us  (min {d.min():.2f} max {d.max():.2f})")
print("softmax-warp entry vs kernel entry: mean %.2f us" % np.mean((h[:, 6] - k[:, 0]) / 1e3))
print("exit (last CTA) from first entry: %.2f us" % kr(5).max())
