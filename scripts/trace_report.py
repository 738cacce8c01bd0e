"""Read Q4_TRACE dumps: per launch, average epilogue phase durations per tile (us)."""
import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
rec = 16 + 148 * 64 * 8 * 8
names = ["wait_tfull", "pass1", "xchg1", "passA", "xchg2", "passB"]
for i in range(len(raw) // rec):
    hdr = np.frombuffer(raw[i * rec:i * rec + 16], np.int32)
    t = np.frombuffer(raw[i * rec + 16:(i + 1) * rec], np.uint64).reshape(148, 64, 8).astype(np.float64)
    grid = hdr[0]
    t = t[:grid]
    ok = (t[:, :, 0] > 0) & (t[:, :, 6] > 0)
    d = {}
    prev = 0
    for k, nm in zip(range(1, 7), names):
        valid = ok & (t[:, :, k] > 0)
        if valid.sum() == 0:
            continue
        # duration from the previous recorded stamp
        pk = t[:, :, prev]
        d[nm] = float(np.mean((t[:, :, k] - pk)[valid]) / 1e3)
        prev = k
    tot = float(np.mean((t[:, :, 6] - t[:, :, 0])[ok]) / 1e3)
    t0 = t[:, :, 0][t[:, :, 0] > 0].min()
    t1 = t[:, :, 6].max()
    print(f"launch kind={hdr[1]} TN={hdr[2]} M={hdr[3]} grid={grid} tiles={int(ok.sum())} "
          f"per-tile {tot:.2f} us: " + " ".join(f"{k}={v:.2f}" for k, v in d.items()) +
          f" | span {(t1 - t0) / 1e3:.1f} us")

# unpack stamps (slot 63 of each CTA): mean ns per k-block
for i in range(len(raw) // rec):
    t = np.frombuffer(raw[i * rec + 16:(i + 1) * rec], np.uint64).reshape(148, 64, 8).astype(np.float64)
    u = t[:, 63, :]
    n = u[:, 4]
    ok = n > 0
    if ok.sum():
        m = (u[ok, :4] / n[ok, None]).mean(0)
        print(f"  unpack per k-block (ns): wait_full_p={m[0]:.0f} wait_empty_u={m[1]:.0f} unpack={m[2]:.0f} fence+arrive={m[3]:.0f}")

# MMA issuer stamps (slot 62): per tile means (us)
for i in range(len(raw) // rec):
    t = np.frombuffer(raw[i * rec + 16:(i + 1) * rec], np.uint64).reshape(148, 64, 8).astype(np.float64)
    u = t[:, 62, :]
    ok = u[:, 3] > 0
    if ok.sum():
        m = (u[ok, :3] / u[ok, 3:4]).mean(0) / 1e3
        print(f"  mma per tile (us): wait_tempty={m[0]:.2f} wait_full_u={m[1]:.2f} issue_span={m[2]:.2f}")
