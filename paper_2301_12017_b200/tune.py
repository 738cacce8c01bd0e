"""Per-part quantization strategy tuner ("different
quantization strategies can be applied given a target scenario and hardware").

The four parts (QKV projection, attention output, MLP intermediate, MLP output) can each
run W4A4 or FP16 (q4_layer_cfg.fp16_parts); for a deployment shape (batch, seq) every one
of the 2^4 strategies is captured as a CUDA graph of the whole encoder and timed on the
device (p50 of `reps` replays), and the fastest is returned.  Strategy names follow the
paper: "qall" = all four quantized, "q3" = only the MLP intermediate quantized, "fp16" =
none quantized, else the quantized parts, e.g. "q1q3".  Marshalling and timing only."""
from __future__ import annotations

import torch

from .encoder import W4A4Encoder

PARTS = ("q1", "q2", "q3", "q4")  # QKV, attention output, MLP intermediate, MLP output


def strategy_name(fp16_parts: int) -> str:
    q = [PARTS[i] for i in range(4) if not fp16_parts >> i & 1]
    return "qall" if len(q) == 4 else ("fp16" if not q else "".join(q))


def time_strategy(cfg: dict, layers: list, B: int, S: int, fp16_parts: int, device="cuda", reps: int = 100,
                  x: torch.Tensor | None = None) -> float:
    """p50 device time (ms) of one captured forward of the encoder under `fp16_parts`."""
    enc = W4A4Encoder(cfg, layers, device=device, fp16_parts=fp16_parts)
    if x is None:
        x = torch.randn(B * S, cfg["hidden"], device=device).half()
    out = torch.empty_like(x)
    enc.capture(x, out, B, S)
    for _ in range(5):
        enc.replay()
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    torch.cuda.synchronize()
    ev[0].record(stream)
    for i in range(reps):
        enc.replay()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    t = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
    del enc
    return t[reps // 2]


def tune(cfg: dict, layers: list, B: int, S: int, device="cuda", reps: int = 100, x=None) -> dict:
    """All 16 strategies at (B, S): {'times': {name: ms}, 'best': name, 'best_fp16_parts': mask}."""
    times, masks = {}, {}
    for m in range(16):
        n = strategy_name(m)
        times[n] = time_strategy(cfg, layers, B, S, m, device, reps, x)
        masks[n] = m
    best = min(times, key=times.get)
    return {"times": times, "best": best, "best_fp16_parts": masks[best]}
