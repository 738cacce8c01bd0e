import sys, numpy as np
raw = np.frombuffer(open(sys.argv[1], "rb").read(), np.uint64).astype(np.float64)
rec = 512 * 16 * 16
t = raw[-rec:].reshape(512, 16, 16)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
t = t[:B]
t0 = min(t[:, :, 0][t[:, :, 0] > 0].min(), t[:, 0, 6][t[:, 0, 6] > 0].min())
start = (t[:, 0, 0] - t0) / 1e3
end = (t[:, 15, 5] - t0) / 1e3
print(f"CTA start: min {start.min():.1f} max {start.max():.1f} us; end: min {end.min():.1f} max {end.max():.1f}; mean duration {np.mean(end - start):.1f}")
hist = np.histogram(start, bins=8)
print("start hist", hist[0].tolist(), np.round(hist[1], 1).tolist())
names = ["wait_S", "softmax", "(gap)", "wait_O", "epilogue"]
d = [np.mean(t[:, 1:15, k + 1] - t[:, 1:15, k]) / 1e3 for k in range(5)]
print("per head us:", " ".join(f"{n}={v:.2f}" for n, v in zip(names, d)))
ent = (t[:, 0, 6] - t0) / 1e3
qe = (t[:, 0, 7] - t0) / 1e3
print(f"softmax-warp entry: min {ent.min():.1f} max {ent.max():.1f}; quantize end: min {qe.min():.1f} max {qe.max():.1f}; "
      f"quantize mean {np.mean(qe - end):.1f} us")
q1 = (t[:, 1, 6] - t0) / 1e3; q2 = (t[:, 1, 7] - t0) / 1e3; q3 = (t[:, 2, 6] - t0) / 1e3
print(f"quantize: barrier wait {np.mean(q1 - end):.2f} first load {np.mean(q2 - q1):.2f} first batch {np.mean(q3 - q2):.2f} rest {np.mean(qe - q3):.2f} us")
a = lambda k0, k1: np.mean(t[:, 3:15, k1] - t[:, 3:15, k0]) / 1e3
print(f"softmax split: ld+max+combine {a(1, 6):.2f} exp loop {a(6, 7):.2f} wait_st+sum combine+arrive {a(7, 2):.2f} us")
print(f"epilogue split: tmem ld {a(4, 8):.2f} pack {a(8, 9):.2f} store {a(9, 5):.2f} us")
