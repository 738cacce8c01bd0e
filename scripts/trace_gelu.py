"""Profiling only: per-tile phase durations of the deferred GELU_Q4 epilogue (Q4_TRACE dump).
Stamps: 0 top, 1 accumulator ready, 2 pass A done (TMEM released), 3 partial published,
4 previous tile's exchange complete, 5 its pass B done, 6 its codes stored + y parked."""
import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
rec = 16 + 148 * 64 * 8 * 8
names = ["wait_acc", "passA", "publish", "xchg_wait", "passB", "store+park"]
for i in range(len(raw) // rec):
    hdr = np.frombuffer(raw[i * rec:i * rec + 16], np.int32)
    if hdr[1] != 2:
        continue
    t = np.frombuffer(raw[i * rec + 16:(i + 1) * rec], np.uint64).reshape(148, 64, 8).astype(np.float64)[:hdr[0]]
    ok = (t[:, 2:62, 0] > 0) & (t[:, 2:62, 6] > 0) & (t[:, 2:62, 4] > 0)
    tt = t[:, 2:62]
    d = {nm: float(np.mean((tt[:, :, k + 1] - tt[:, :, k])[ok]) / 1e3) for k, nm in enumerate(names)}
    per = float(np.mean((tt[:, 1:, 0] - tt[:, :-1, 0])[ok[:, 1:] & ok[:, :-1]]) / 1e3)
    print(f"kind={hdr[1]} TN={hdr[2]} M={hdr[3]} grid={hdr[0]} tile period {per:.2f} us: " +
          " ".join(f"{k}={v:.2f}" for k, v in d.items()))
