"""Measured INT8 tensor-core ceiling on this B200: cuBLASLt int8 x int8 ->
int32 through torch._int_mm at 8192^3, as a burst (best of 10 single launches) and sustained
(back to back for 4 s, the power-capped rate a kernel inside a long step sees), with the SM
clocks sampled by nvidia-smi during each phase.  Writes one JSON object to stdout (and to the
path given as argv[1], if any)."""
import json
import statistics
import subprocess
import sys
import time

import torch


def clocks_during(fn):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.sw_power_cap,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100", "-i", "0"],
                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    time.sleep(0.3)
    r = fn()
    time.sleep(0.2)
    p.terminate()
    out = p.communicate(timeout=5)[0]
    sm, cap = [], 0
    for line in out.splitlines():
        f = [x.strip() for x in line.split(",")]
        try:
            sm.append(float(f[0]))
            cap += f[1].lower() == "active"
        except (ValueError, IndexError):
            pass
    load = [s for s in sm if sm and s > 0.5 * max(sm)] or sm
    return r, {"sm_mhz_median": statistics.median(load) if load else None, "samples": len(sm),
               "sw_power_cap_samples": cap}


def main():
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(42)
    a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
    w = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
    b = w.t()  # [K, N] column-major view: the TN layout cuBLASLt runs on the int8 tensor cores
    ops = 2.0 * n ** 3
    for _ in range(5):
        torch._int_mm(a, b)
    torch.cuda.synchronize()

    def burst():
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            time.sleep(0.05)
        return ops / (min(ts) * 1e-3) / 1e12

    def sustained():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 0
        t_end = time.time() + 4.0
        e0.record()
        while time.time() < t_end:
            for _ in range(20):
                torch._int_mm(a, b)
            k += 20
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        return ops * k / (e0.elapsed_time(e1) * 1e-3) / 1e12

    tb, cb = clocks_during(burst)
    ts, cs = clocks_during(sustained)
    r = {"what": "torch._int_mm int8 x int8 -> int32 (cuBLASLt), M = N = K = 8192, ops = 2 N^3",
         "int8_tops_burst": tb, "clocks_burst": cb, "int8_tops_sustained": ts, "clocks_sustained": cs,
         "gpu": torch.cuda.get_device_name(0), "torch": torch.__version__}
    s = json.dumps(r)
    print(s)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(s + "\n")


if __name__ == "__main__":
    main()
