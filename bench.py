#!/usr/bin/env python
"""bench.py -- W4A4 BERT encoder throughput on B200 (BASELINE.json configs[3]):
BERT-large, 24 layers, global batch 256, seq 128, all four linears W4A4 ("qall"),
batch-sharded data parallel over N GPUs (strong scaling at the fixed global
batch of 256 -- rank r runs sequences [r*256/N, (r+1)*256/N) -- with weak scaling, 256
sequences per GPU, measured as a secondary figure; no collective in the data path beyond
the NCCL all-gather of the outputs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N ... bench.py --gpus N ...

With --gpus N > 1 and no torchrun environment, bench.py launches itself under
torch.distributed.run with N ranks (127.0.0.1); under torchrun, WORLD_SIZE must equal N.

One step = one pass of the whole hot path: initial activation
quantize + 24 x [QKV W4A4 GEMM, FP16 attention + ctx quantize, attn-out W4A4 GEMM +
residual/LN/requant, FFN1 W4A4 GEMM + GELU/requant, FFN2 W4A4 GEMM + residual/LN/requant]
over 256 x 128 tokens per GPU, replayed as one CUDA graph with inputs resident in HBM.
Rank 0 prints ONE JSON line (keys documented in DESIGN.md "Measurement")."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
WORKLOAD = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"][3]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="large", choices=["base", "large"])
    ap.add_argument("--batch", type=int, default=256,
                    help="global batch (strong scaling) or sequences per GPU (--scaling weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: fixed global batch (strong, SURVEY 8(e) primary) or fixed per-GPU batch")
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--layers", type=int, default=0, help="0 = the model's own depth")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip latency / GEMM side measurements")
    ap.add_argument("--gather", default="cls", choices=["cls", "full", "none"],
                    help="N>1: NCCL all-gather of the outputs inside every timed step (SURVEY 8(e))")
    ap.add_argument("--oracle-worker", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-launch this script as N ranks."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", ",".join(str(g) for g in self.gpus)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out = self.p.communicate(timeout=5)[0]
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def peaks():
    p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = p.get("hbm_gbs", 6650.0)
    bf16 = p.get("bf16_tflops_sustained", 1400.0)
    bf16b = p.get("bf16_tflops", 1636.0)
    src = "measured" if p else "fallback"
    # dense INT8 = 2 x dense bf16 nominal (4.5 vs 2.25 POPS); applied to the measured bf16 figures:
    # sustained for a kernel inside the long step, burst for a kernel timed alone (GEMM sweep)
    return {"hbm_gbs": hbm, "int8_tops": 2.0 * bf16, "int8_tops_burst": 2.0 * bf16b, "bf16_tflops": bf16,
            "source": src}


def gemm_work(M, N, K, kind):
    """Algorithmic ops and bytes of one W4A4 linear launch."""
    ops = 2.0 * M * N * K
    by = M * K / 2 + N * K / 2 + 4 * M + 4 * N + 2 * N  # A codes, W codes, scales, bias
    if kind == "f16":
        by += 2.0 * M * N
    elif kind == "gelu_q4":
        by += M * N / 2 + 4 * M
    elif kind == "resln_q4":
        by += 2.0 * M * N + 4 * N + 2.0 * M * N + M * N / 2 + 4 * M  # residual, gamma/beta, f16 out, codes
    return ops, by


def attention_work(B, S, H, d=64):
    h = H * d
    ops = 4.0 * B * H * S * S * d
    by = B * S * 3 * h * 2 + B * S * h / 2 + 4 * B * S  # qkv in, codes + scales out
    return ops, by


# ----------------------------------------------------------------------------- reference arm
_ORACLE_W = {}


def _oracle_layer_weights(orc, synth, cfg, layer=0, threads=0):
    key = (cfg["hidden"], cfg["ffn"], layer)
    if key not in _ORACLE_W:
        p = synth.layer_params(cfg, layer, "bert")
        w = dict(p)
        for k in ("wqkv", "wo", "w1", "w2"):
            w[k], w["s" + k[1:]] = orc.quantize_rows(p[k], threads=threads)
        _ORACLE_W[key] = w
    return _ORACLE_W[key]


def oracle_sample(cfg, n_seq, S, threads=0, layers=1):
    """Time the CPU oracle (as it stands) on `layers` encoder layers over n_seq sequences:
    the initial quantize + L x O-9.  Weight generation / quantization (offline in the
    product path too) is not timed."""
    import numpy as np
    import oracle as orc
    from paper_2301_12017_b200 import synth
    ws = [_oracle_layer_weights(orc, synth, cfg, l, threads) for l in range(layers)]
    x = np.concatenate([synth.hidden(S, cfg["hidden"], "input", b) for b in range(n_seq)])
    t0 = time.perf_counter()
    xq, xs = orc.quantize_rows(x, threads=threads)
    for w in ws:
        o = orc.encoder_layer(cfg, w, n_seq, S, x, xq, xs, threads=threads)
        x, xq, xs = o["h_out"], o["hq_out"], o["hs_out"]
    return time.perf_counter() - t0


def oracle_linear_sample(M, N, K, threads=0):
    """BASELINE configs[0]: one W4A4 linear (F16 epilogue) through the oracle."""
    import oracle as orc
    from paper_2301_12017_b200 import synth
    x = synth.hidden(M, K, "c1_x")
    w = synth.layer_params(synth.BERT["base"], 0, "bert")["wo"]
    wc, wsc = orc.quantize_rows(w, threads=threads)
    t0 = time.perf_counter()
    xc, xsc = orc.quantize_rows(x, threads=threads)
    orc.w4a4_linear(xc, xsc, wc, wsc, M, N, K, orc.EPI_F16, threads=threads)
    return time.perf_counter() - t0


def oracle_worker(spec: str) -> int:
    """Child process of the cpu_baseline leg: time the oracle, print one JSON object.
    Runs apart from the product process, so the GPU arm never loads liboracle.so."""
    from paper_2301_12017_b200 import synth
    sp = json.loads(spec)
    out = {}
    large, base = dict(synth.BERT["large"]), dict(synth.BERT["base"])
    th_all = cpu_cores()  # explicit: torchrun exports OMP_NUM_THREADS=1
    # BASELINE configs[3] slice: one BERT-large layer over 16 sequences (M = 2048),
    # all host threads; and a 1-thread run on a 2-sequence slice
    t = [oracle_sample(large, 16, 128, th_all) for _ in range(sp.get("reps", 2))]
    out["large_layer_m2048_s"] = statistics.median(t)
    out["large_layer_m256_1thread_s"] = oracle_sample(large, 2, 128, 1)
    if sp.get("configs", True):
        # configs[0..2] timed in full: linear M=128 K=N=768; BERT-base layer bs 1; 12 layers bs 1
        out["c1_linear_m128_s"] = statistics.median(oracle_linear_sample(128, 768, 768) for _ in range(5))
        out["c2_base_layer_bs1_s"] = statistics.median(oracle_sample(base, 1, 128, th_all) for _ in range(5))
        out["c3_base_12layer_bs1_s"] = statistics.median(oracle_sample(base, 1, 128, th_all, 12) for _ in range(2))
    print(json.dumps(out), flush=True)
    return 0


def cpu_baseline_subprocess(L: int, reps: int = 2):
    """cpu_baseline of our arm (rank 0, N=1): the oracle timed in a child process."""
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--oracle-worker",
                        json.dumps({"reps": reps})], capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        raise RuntimeError(f"oracle worker failed: {r.stderr[-2000:]}")
    o = json.loads(r.stdout.strip().splitlines()[-1])
    t = o["large_layer_m2048_s"]
    return {"value": 16 / (t * L), "unit": "seq/s", "cores": cpu_cores(), "kind": "oracle",
            "sample": f"1 BERT-large layer x 16 seq x 128 tok (M = 2048, one slice of the workload), "
                      f"median of {reps}, all host threads, extrapolated x{L} layers (x16 slices = the "
                      f"256-seq batch at the same seq/s)",
            "one_thread_seq_per_s": 2 / (o["large_layer_m256_1thread_s"] * L),
            "configs_full_s": {k: v for k, v in o.items() if k.startswith("c")}}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # under torchrun only rank 0 runs the CPU oracle
    from paper_2301_12017_b200 import synth
    cfg = dict(synth.BERT[args.model])
    L = args.layers or cfg["layers"]
    cores = cpu_cores()
    n_seq = 16  # one M = 2048 slice of the batch per step
    times = []
    for i in range(args.warmup + args.steps):
        t = oracle_sample(cfg, n_seq, args.seq, threads=cores)  # explicit: torchrun sets OMP_NUM_THREADS=1
        if i >= args.warmup:
            times.append(t)
    t = statistics.median(times)
    value = n_seq / (t * L)  # seq/s of the full L-layer encoder (layers are identical work)
    sample = (f"1 {args.model} encoder layer x {n_seq} seq x {args.seq} tok (M = {n_seq * args.seq}) per step, "
              f"all host threads, extrapolated x{L} layers")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "seq/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": args.scaling if args.gpus > 1 else "strong", "vs_baseline": None,
            "dtype": "int64/f64 (CPU oracle)", "data": "synthetic",
            "config": {"workload": WORKLOAD, "model": f"bert-{args.model}", "layers": L,
                       "global_batch": args.batch, "seq_len": args.seq},
            "cpu_baseline": {"value": value, "unit": "seq/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "seq/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.oracle_worker is not None:
        return oracle_worker(args.oracle_worker)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2301_12017_b200 as q4
    from paper_2301_12017_b200 import synth

    from paper_2301_12017_b200 import dist as qd

    rank, world, local = qd.env_ranks()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N = world
    barrier = qd.barrier

    def max_over_ranks(x: float) -> float:
        return qd.max_over_ranks(x, dev)

    cfg = dict(synth.BERT[args.model])
    L = args.layers or cfg["layers"]
    S, h = args.seq, cfg["hidden"]
    GB = args.batch if args.scaling == "strong" else args.batch * N  # global batch
    if GB % N:
        raise SystemExit(f"bench.py: global batch {GB} does not split evenly over {N} ranks")
    start, B = qd.shard(GB, rank, N)  # this rank's contiguous slice of the global batch
    M = B * S
    layers = [synth.layer_params(cfg, l, "bert") for l in range(L)]
    enc = q4.W4A4Encoder(cfg, layers, device=dev)
    del layers
    x = np.concatenate([synth.hidden(S, h, "input", b) for b in range(start, start + B)])
    xd = torch.from_numpy(x).to(dev)
    out = torch.empty_like(xd)

    # kernels per step (counted through the library, one eager forward)
    n0 = q4.launch_count()
    enc.forward(xd, out, B, S)
    torch.cuda.synchronize()
    launches_per_step = q4.launch_count() - n0

    enc.capture(xd, out, B, S)
    stream = torch.cuda.current_stream()
    # the one data collective (N > 1): gather the outputs of every rank after the last layer
    gather = qd.OutputGather(B, S, h, args.gather, dev) if (world > 1 and args.gather != "none") else None

    def step():
        enc.replay()
        if gather is not None:
            gather(out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ------------------------------------------------------------------ timed region
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(list(range(N)) if rank == 0 else [local]) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = ev[0].elapsed_time(ev[-1])
    ms_per_step = max_over_ranks(total_ms / args.steps)
    p50 = max_over_ranks(statistics.median(step_ms))
    value = GB / (ms_per_step / 1e3)
    clocks = clk.summary()
    gather_info = None
    if gather is not None:
        # both gather modes timed alone on the same stream (device time, max over ranks)
        gather_info = {"in_step": args.gather, "bytes_per_rank": gather.bytes_per_rank}
        for mode in ("cls", "full"):
            g = qd.OutputGather(B, S, h, mode, dev)
            g(out)
            torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(10):
                g(out)
            b.record(stream)
            torch.cuda.synchronize()
            gather_info[f"{mode}_ms"] = max_over_ranks(a.elapsed_time(b) / 10)
            gather_info[f"{mode}_bytes_per_rank"] = g.bytes_per_rank
            del g

    # ------------------------------------------------------------------ end to end (host buffers)
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(x).pin_memory()
        oh = torch.empty(xh.shape, dtype=torch.float16).pin_memory()
        for _ in range(max(1, args.warmup)):
            enc.forward(xh, oh, B, S)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            enc.forward(xh, oh, B, S)  # H2D copy + L layers + D2H copy, all in the C call
        e1.record(stream)
        torch.cuda.synchronize()
        serial_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        ok = torch.equal(oh, out.cpu())
        # pipelined serving (q4_encoder_pipeline): every step still uploads its input from
        # pinned host memory and downloads its output, overlapped with the neighbouring
        # steps' forward passes (two pinned host buffers per direction, cycled)
        xs_h = [xh, torch.from_numpy(x).pin_memory()]
        os_h = [torch.empty_like(oh).pin_memory() for _ in range(2)]
        ins = [xs_h[i % 2] for i in range(args.steps)]
        outs = [os_h[i % 2] for i in range(args.steps)]
        enc.serve(ins[:2], outs[:2], B, S)
        torch.cuda.synchronize()
        barrier()
        e0.record(stream)
        enc.serve(ins, outs, B, S)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        ok = ok and torch.equal(os_h[(args.steps - 1) % 2], out.cpu())
        e2e = {"value": GB / (e2e_ms / 1e3), "unit": "seq/s", "h2d_bytes_per_step": M * h * 2,
               "d2h_bytes_per_step": M * h * 2, "ms_per_step": e2e_ms, "matches_device_path": ok,
               "api": "W4A4Encoder.serve -> q4_encoder_pipeline (copies overlapped across steps)",
               "serial_ms_per_step": serial_ms, "serial_value": GB / (serial_ms / 1e3)}

    # ------------------------------------------------------------------ per-kernel breakdown
    # One instrumented forward: the same launches as the graph, issued one by one with CUDA
    # events on the launching stream around each, averaged over the L layers.
    pk = peaks()
    kinds = {}
    w0 = enc.weights
    hq, hs = q4.quantize_rows(xd)
    hcur = xd
    f = cfg["ffn"]

    def timed(name, fn, work):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = fn()
        b.record(stream)
        kinds.setdefault(name, {"events": [], "work": work})["events"].append((a, b))
        return r

    for rep in range(2):  # pass 0 warms the caching allocator; pass 1 is measured
        kinds.clear()
        hq, hs = q4.quantize_rows(xd)
        hcur = xd
        for l in range(L):
            w = w0[l]
            qkv = timed("qkv_gemm_f16", lambda: q4.w4a4_linear(
                hq, hs, w["wqkv"], w["sqkv"], q4.EPI_F16, bias=w["bqkv"], w_i8=w.get("wqkv8")),
                gemm_work(M, 3 * h, h, "f16"))["f16"]
            cq, cs = timed("attention_q4", lambda: q4.attention_f16_q4(qkv, B, S, cfg["heads"]),
                           attention_work(B, S, cfg["heads"]))
            o1 = timed("attn_out_gemm_resln_q4", lambda: q4.w4a4_linear(
                cq, cs, w["wo"], w["so"], q4.EPI_RESLN_Q4, bias=w["bo"], residual=hcur,
                gamma=w["ln1_g"], beta=w["ln1_b"], w_i8=w.get("wo8")), gemm_work(M, h, h, "resln_q4"))
            o2 = timed("ffn1_gemm_gelu_q4", lambda: q4.w4a4_linear(
                o1["codes"], o1["scales"], w["w1"], w["s1"], q4.EPI_GELU_Q4, bias=w["b1"],
                w_i8=w.get("w18")), gemm_work(M, f, h, "gelu_q4"))
            o3 = timed("ffn2_gemm_resln_q4", lambda: q4.w4a4_linear(
                o2["codes"], o2["scales"], w["w2"], w["s2"], q4.EPI_RESLN_Q4, bias=w["b2"],
                residual=o1["f16"], gamma=w["ln2_g"], beta=w["ln2_b"], w_i8=w.get("w28")),
                gemm_work(M, h, f, "resln_q4"))
            hcur, hq, hs = o3["f16"], o3["codes"], o3["scales"]
        torch.cuda.synchronize()
    breakdown = {}
    for name, d in kinds.items():
        t = statistics.median(a.elapsed_time(b) for a, b in d["events"])  # ms per launch
        ops, by = d["work"]
        breakdown[name] = {"ms": t, "TOPS": ops / (t * 1e-3) / 1e12, "GBps": by / (t * 1e-3) / 1e9,
                           "ops": ops, "bytes": by}
    step_sum = sum(v["ms"] for v in breakdown.values()) * L
    for v in breakdown.values():
        v["share"] = v["ms"] * L / step_sum
    dom = max(breakdown, key=lambda k: breakdown[k]["ms"])
    d = breakdown[dom]
    ridge = pk["int8_tops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    if d["ops"] / d["bytes"] > ridge and "gemm" in dom:
        roof = {"bound": "tensor", "achieved": d["TOPS"], "peak": pk["int8_tops"], "unit": "TOPS",
                "frac": d["TOPS"] / pk["int8_tops"]}
    else:
        roof = {"bound": "hbm", "achieved": d["GBps"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": d["GBps"] / pk["hbm_gbs"]}
    roof.update({"kernel": dom, "traffic": None, "share_of_step": d["share"],
                 "peak_source": f"{pk['source']}: " + ("2 x bf16_tflops_sustained (int8 = 2x bf16 nominal)"
                                                       if roof["bound"] == "tensor" else "hbm_gbs")})
    ic = os.path.join(ROOT, "profiles", "r2", "int8_ceiling.json")
    if os.path.exists(ic) and roof["bound"] == "tensor":
        c = json.load(open(ic))
        roof["int8_ceiling_measured"] = {"burst_tops": c.get("int8_tops_burst"), "sustained_tops": c.get("int8_tops_sustained"),
                                         "how": c.get("what"), "sustained_sm_mhz": c.get("clocks_sustained", {}).get("sm_mhz_median")}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tr = json.load(open(tp)).get(f"{args.model}:{dom}:M{M}")
        if tr:
            roof["traffic"] = tr

    # ------------------------------------------------------------------ extras (rank 0, N=1 shapes)
    extras = {}
    if not args.no_extras and rank == 0:
        extras = side_measurements(q4, synth, torch, np, dev, args)
        if N == 1:
            extras["strong_scaling_model"] = strong_scaling_model(enc, synth, torch, np, dev, args, ms_per_step)

    # ------------------------------------------------------------------ weak scaling (N > 1, secondary)
    weak = None
    if N > 1 and args.scaling == "strong":
        # 256 sequences per rank (the global batch grows with N): same graph at M = 256 * S
        Bw = args.batch
        sw0, _ = qd.shard(Bw * N, rank, N)
        xw = torch.from_numpy(np.concatenate([synth.hidden(S, h, "input", b) for b in range(sw0, sw0 + Bw)])).to(dev)
        ow = torch.empty_like(xw)
        encw = enc.sibling()
        encw.capture(xw, ow, Bw, S)
        gw = qd.OutputGather(Bw, S, h, args.gather, dev) if args.gather != "none" else None
        for _ in range(args.warmup):
            encw.replay()
            if gw is not None:
                gw(ow)
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            encw.replay()
            if gw is not None:
                gw(ow)
        b.record(stream)
        torch.cuda.synchronize()
        wms = max_over_ranks(a.elapsed_time(b) / args.steps)
        weak = {"value": Bw * N / (wms / 1e3), "unit": "seq/s", "ms_per_step": wms, "batch_per_gpu": Bw,
                "global_batch": Bw * N}
        del encw, xw, ow, gw

    # ------------------------------------------------------------------ CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_subprocess(L)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "seq/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "p50_ms": p50, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int4 (W4A4, s8 tensor-core MMA, s32 acc)",
            "data": "synthetic (seeded, random-init weights)",
            "config": {"workload": WORKLOAD, "model": f"bert-{args.model}", "layers": L, "batch_per_gpu": B,
                       "global_batch": GB, "seq_len": S, "parallelism": f"dp{N} (batch-sharded replicas" + (
                           f", NCCL all-gather of the {args.gather} outputs per step)" if gather is not None else ", no collective)"),
                       "l2": f"no flush: per-step working set {(M * h * 2 * 6 + M * cfg['ffn'] / 2) / 1e9:.2f} GB "
                             f"of activations + {sum(v.numel() for w in enc.weights for v in w.values()) / 1e6:.0f} MB "
                             f"weights >> 126 MB L2", "cuda_graph": True},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks, "gather": gather_info, "weak_scaling": weak, "kernels": breakdown, "extras": extras, "lib": q4.version(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def strong_scaling_model(enc, synth, torch, np, dev, args, ms_n1):
    """SURVEY 8(e) on one GPU: the per-rank step of an N-way strong-scaled run is this model at
    batch 256/N (M = 16384 / 8192 / 4096).  Predicted N-GPU seq/s = 256 / t(256/N), before
    the [CLS] gather (0.5 MB; NCCL is not measurable on one GPU)."""
    S, h = args.seq, enc.cfg["hidden"]
    stream = torch.cuda.current_stream()
    out = {"n1_ms": ms_n1}
    for n in (2, 4, 8):
        B = args.batch // n
        x = torch.from_numpy(np.concatenate([synth.hidden(S, h, "input", b) for b in range(B)])).to(dev)
        o = torch.empty_like(x)
        e = enc.sibling()
        e.capture(x, o, B, S)
        for _ in range(5):
            e.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(20):
            e.replay()
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 20
        out[f"n{n}"] = {"batch_per_gpu": B, "M": B * S, "ms": t, "pred_seq_per_s": args.batch / (t * 1e-3),
                        "pred_efficiency": ms_n1 / (n * t)}
        del e, x, o
    return out


def side_measurements(q4, synth, torch, np, dev, args):
    """Latency configs (BASELINE configs[1], [2]), the FFN GEMM TOPS (configs[4]) and the
    W8A8 baseline (encoder and GEMM at 8 bits, same kernels)."""
    out = {}
    stream = torch.cuda.current_stream()
    base = dict(synth.BERT["base"])
    for L, name in ((1, "bert_base_1layer_bs1_p50_ms"), (12, "bert_base_12layer_bs1_p50_ms")):
        enc = q4.W4A4Encoder(base, [synth.layer_params(base, l, "bert") for l in range(L)], device=dev)
        x = torch.from_numpy(synth.hidden(128, 768, "input", 0)).to(dev)
        o = torch.empty_like(x)
        enc.capture(x, o, 1, 128)
        for _ in range(20):
            enc.replay()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(201)]
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(200):
            enc.replay()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(200))
        out[name] = t[100]
        out[name.replace("p50", "p10")] = t[20]
        out[name.replace("p50", "p90")] = t[180]
        # cold L2: a 256 MB write (> the 126 MB L2) before every replay, timed outside the pair
        # of events around the replay, so weights and activations come from HBM each time
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(100)]
        ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(100)]
        for i in range(100):
            flush.fill_(i & 0xFF)
            ev0[i].record(stream)
            enc.replay()
            ev1[i].record(stream)
        torch.cuda.synchronize()
        t = sorted(ev0[i].elapsed_time(ev1[i]) for i in range(100))
        out[name.replace("bs1_p50", "bs1_cold_l2_p50")] = t[50]
        del flush
    # configs[0]: one W4A4 linear, M = 128 (batch 1 x seq 128), K = N = 768, fp16 out (and the
    # fused residual + LayerNorm + requant epilogue of the same shape), prepacked weights; a CUDA
    # graph of one launch replayed, p50 of 200 (the floor of one launch in a graph: 1 empty kernel)
    Mq, Kq, Nq = 128, 768, 768
    xq = torch.from_numpy(synth.hidden(Mq, Kq, "c1x")).to(dev)
    aq, saq = q4.quantize_rows(xq)
    wq, swq = q4.quantize_rows(torch.from_numpy(synth.weight(Nq, Kq, "c1w")).to(dev))
    w8q = q4.prepack_weights(wq)
    bq = torch.from_numpy(synth.bias(Nq, "c1b")).to(dev)
    resq = torch.from_numpy(synth.hidden(Mq, Nq, "c1r")).to(dev)
    gq = torch.ones(Nq, dtype=torch.float16, device=dev)
    for kind, nm, kw in ((q4.EPI_F16, "config1_linear_m128_k768_n768_f16_p50_us", {}),
                         (q4.EPI_RESLN_Q4, "config1_linear_m128_k768_n768_resln_q4_p50_us",
                          dict(residual=resq, gamma=gq, beta=bq))):
        wsq = torch.zeros(max(q4.lib().q4_w4a4_linear_workspace(Mq, Nq, Kq, kind), 1), dtype=torch.uint8, device=dev)
        oq = q4.w4a4_linear(aq, saq, wq, swq, kind, bias=bq, w_i8=w8q, workspace=wsq, **kw)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            q4.w4a4_linear(aq, saq, wq, swq, kind, bias=bq, w_i8=w8q, workspace=wsq, out=oq, **kw)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            q4.w4a4_linear(aq, saq, wq, swq, kind, bias=bq, w_i8=w8q, workspace=wsq, out=oq, **kw)
        for _ in range(20):
            g.replay()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(201)]
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(200):
            g.replay()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(200))
        out[nm] = t[100] * 1e3
    # Latency floor (SURVEY 8(d) configs[2]): a CUDA graph of as many empty PDL kernels as the
    # 12-layer bs-1 forward launches (1 + 12 x 5), same launch attributes, p50 of 200 replays
    for nk, nm in ((61, "latency_floor_61_empty_kernels_ms"), (6, "latency_floor_6_empty_kernels_ms"),
                   (1, "latency_floor_1_empty_kernel_ms")):
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            q4.launch_floor(nk, 36)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            q4.launch_floor(nk, 36)
        for _ in range(20):
            g.replay()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(201)]
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(200):
            g.replay()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(200))
        out[nm] = t[100]
    # The paper's INT4-vs-INT8 comparison (Fig. e2e_i4_i8): the W8A8
    # baseline encoder (same kernels at 8 bits) on the bench workload and the latency config
    for size, L, B, name in (("large", 24, 256, "w8a8_bert_large_24l_bs256"), ("base", 12, 1, "w8a8_bert_base_12l_bs1")):
        c = dict(synth.BERT[size])
        enc = q4.W8A8Encoder(c, [synth.layer_params(c, l, "bert") for l in range(L)], device=dev)
        x = torch.from_numpy(np.concatenate([synth.hidden(128, c["hidden"], "input", b) for b in range(B)])).to(dev)
        o = torch.empty_like(x)
        enc.capture(x, o, B, 128)
        for _ in range(5):
            enc.replay()
        n = 20 if B > 1 else 200
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(n):
            enc.replay()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(n))
        out[name + "_p50_ms"] = t[n // 2]
        out[name + "_seq_per_s"] = B / (t[n // 2] * 1e-3)
        del enc
    # Asymmetric activations (NEXT-3; the paper finds asym slower "because of less required
    # computation for bias term"): the same encoder with asym_acts = 1
    for size, L, B, name in (("large", 24, 256, "asym_bert_large_24l_bs256"), ("base", 12, 1, "asym_bert_base_12l_bs1")):
        c = dict(synth.BERT[size])
        enc = q4.W4A4Encoder(c, [synth.layer_params(c, l, "bert") for l in range(L)], device=dev, asym=True)
        x = torch.from_numpy(np.concatenate([synth.hidden(128, c["hidden"], "input", b) for b in range(B)])).to(dev)
        o = torch.empty_like(x)
        enc.capture(x, o, B, 128)
        for _ in range(5):
            enc.replay()
        n = 20 if B > 1 else 200
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(n):
            enc.replay()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        t = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(n))
        out[name + "_p50_ms"] = t[n // 2]
        out[name + "_seq_per_s"] = B / (t[n // 2] * 1e-3)
        del enc
    # Per-part quantization strategy tuner (Fig. e2e_i4_fti8 annotations):
    # all 16 strategies of BERT-base 12 L at the paper's small (bs-seq) points and the
    # latency config; argmin reported with the qall and all-FP16 times
    from paper_2301_12017_b200 import tune
    base12 = [synth.layer_params(base, l, "bert") for l in range(12)]
    for (B, S) in ((1, 32), (8, 32), (1, 128)):
        x = torch.from_numpy(np.concatenate([synth.hidden(S, 768, "input", b) for b in range(B)])).to(dev)
        r = tune.tune(base, base12, B, S, device=dev, reps=50, x=x)
        out[f"strategy_bert_base_12l_bs{B}_seq{S}"] = {"best": r["best"], "best_ms": r["times"][r["best"]],
                                                       "qall_ms": r["times"]["qall"], "fp16_ms": r["times"]["fp16"],
                                                       "q3_ms": r["times"]["q3"], "times": r["times"]}
    # GEMM TOPS at the BERT-large FFN shapes, M = 32768 (tcgen05 vs legacy mma.sync); each GEMM
    # is timed alone, so its fraction is against the burst INT8 peak
    pk = peaks()
    out["gemm_peak_int8_tops_burst"] = pk["int8_tops_burst"]
    for (Nn, K) in ((4096, 1024), (1024, 4096)):
        M = 32768
        a = torch.from_numpy(synth.random_packed(M, K, f"sw_a{K}")).to(dev)
        w = torch.from_numpy(synth.random_packed(Nn, K, f"sw_w{Nn}")).to(dev)
        sa = torch.from_numpy(synth.random_scales(M, "sw_sa")).to(dev)
        sw = torch.from_numpy(synth.random_scales(Nn, "sw_sw")).to(dev)
        a8 = torch.from_numpy(synth.random_i8(M, K, f"sw_a8{K}")).to(dev)
        w8 = torch.from_numpy(synth.random_i8(Nn, K, f"sw_w8{Nn}")).to(dev)
        o = q4.w8a8_linear(a8, sa, w8, sw, q4.EPI_F16)
        for _ in range(3):
            q4.w8a8_linear(a8, sa, w8, sw, q4.EPI_F16, out=o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            q4.w8a8_linear(a8, sa, w8, sw, q4.EPI_F16, out=o)
        e1.record(stream)
        torch.cuda.synchronize()
        tops = 2.0 * M * Nn * K / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12
        out[f"gemm_f16_M{M}_N{Nn}_K{K}_w8a8_tcgen05_TOPS"] = tops
        out[f"gemm_f16_M{M}_N{Nn}_K{K}_w8a8_tcgen05_frac_int8_peak"] = tops / pk["int8_tops_burst"]
        # symmetric vs asymmetric activations (NEXT-3), prepacked weights, F16 epilogue
        w8p = q4.prepack_weights(w)
        xa = torch.from_numpy(synth.hidden(M, K, f"sw_asym{K}") + np.float16(0.5)).to(dev)
        ac, asc, az = q4.quantize_rows_asym(xa)
        wsum = q4.weight_code_sums(w)
        for nm, fn in (("w8_sym", lambda o: q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, w_i8=w8p, out=o)),
                       ("w8_asym", lambda o: q4.w4a4_asym_linear(ac, asc, az, w, sw, wsum, q4.EPI_F16, w_i8=w8p,
                                                                  out=o))):
            o = fn(None)
            for _ in range(3):
                fn(o)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                fn(o)
            e1.record(stream)
            torch.cuda.synchronize()
            out[f"gemm_f16_M{M}_N{Nn}_K{K}_tcgen05_{nm}_TOPS"] = 2.0 * M * Nn * K / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12
        for ml, mname in ((1, "tcgen05"), (2, "mma_sync_s8"), (3, "mma_sync_s4")):
            o = q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, mainloop=ml)
            for _ in range(3):
                q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, mainloop=ml, out=o)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                q4.w4a4_linear(a, sa, w, sw, q4.EPI_F16, mainloop=ml, out=o)
            e1.record(stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 10
            tops = 2.0 * M * Nn * K / (t * 1e-3) / 1e12
            out[f"gemm_f16_M{M}_N{Nn}_K{K}_{mname}_TOPS"] = tops
            out[f"gemm_f16_M{M}_N{Nn}_K{K}_{mname}_frac_int8_peak"] = tops / pk["int8_tops_burst"]
    return out


if __name__ == "__main__":
    sys.exit(main())
