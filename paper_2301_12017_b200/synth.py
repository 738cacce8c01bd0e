"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the tests, ``bench.py`` and ``smoke()``; it feeds BOTH the
CUDA path and the CPU oracle the identical host arrays.  It holds random numbers
only -- none of the method's arithmetic (no quantization, no GEMM, no epilogue).

Recipe:
  * per-tensor seed = crc32(name, layer) mixed with the base seed 42 (PAPER.md:532
    uses seed 42 for its runs); numpy PCG64.
  * hidden input: fp16 N(0,1) x per-token magnitude exp(N(0, 0.5^2)); 1% of tokens
    x8 (per-token spread, "positional activation range").
  * weights: fp16 N(0, 0.02^2) (BERT initializer_range); biases N(0, 0.02^2);
    LayerNorm gamma = 1 + N(0, 0.1^2), beta = N(0, 0.1^2).
  * GEMM-sweep operands: uniformly random INT4 nibbles in [-7, 7] (never all-zero),
    scales uniform in [0.5, 1.5] * 1/16.
"""
from __future__ import annotations

import zlib

import numpy as np

BASE_SEED = 42

# BERT dimensions (PAPER.md:435 gives h = 768 / 1024; heads of 64, 4h FFN, L = 12 / 24)
BERT = {
    "base": dict(hidden=768, heads=12, head_dim=64, ffn=3072, layers=12, ln_eps=1e-12),
    "large": dict(hidden=1024, heads=16, head_dim=64, ffn=4096, layers=24, ln_eps=1e-12),
}


def rng(name: str, layer: int = 0, base: int = BASE_SEED) -> np.random.Generator:
    s = zlib.crc32(f"{name}/{layer}".encode()) ^ (base * 0x9E3779B1)
    return np.random.Generator(np.random.PCG64(s & 0xFFFFFFFFFFFFFFFF))


def hidden(M: int, h: int, name: str = "hidden", layer: int = 0) -> np.ndarray:
    g = rng(name, layer)
    x = g.standard_normal((M, h), dtype=np.float32)
    mag = np.exp(g.standard_normal(M, dtype=np.float32) * 0.5)
    outl = g.random(M) < 0.01
    mag[outl] *= 8.0
    return (x * mag[:, None]).astype(np.float16)


def weight(N: int, K: int, name: str, layer: int = 0) -> np.ndarray:
    return (rng(name, layer).standard_normal((N, K), dtype=np.float32) * 0.02).astype(np.float16)


def bias(N: int, name: str, layer: int = 0) -> np.ndarray:
    return (rng(name, layer).standard_normal(N, dtype=np.float32) * 0.02).astype(np.float16)


def ln_params(N: int, name: str, layer: int = 0):
    g = rng(name, layer)
    gamma = (1.0 + 0.1 * g.standard_normal(N, dtype=np.float32)).astype(np.float16)
    beta = (0.1 * g.standard_normal(N, dtype=np.float32)).astype(np.float16)
    return gamma, beta


def layer_params(cfg: dict, layer: int, prefix: str = "bert"):
    """fp16 parameters of one encoder layer (nn.Linear [out, in] orientation)."""
    h, f = cfg["hidden"], cfg["ffn"]
    p = {
        "wqkv": weight(3 * h, h, f"{prefix}.wqkv", layer),
        "wo": weight(h, h, f"{prefix}.wo", layer),
        "w1": weight(f, h, f"{prefix}.w1", layer),
        "w2": weight(h, f, f"{prefix}.w2", layer),
        "bqkv": bias(3 * h, f"{prefix}.bqkv", layer),
        "bo": bias(h, f"{prefix}.bo", layer),
        "b1": bias(f, f"{prefix}.b1", layer),
        "b2": bias(h, f"{prefix}.b2", layer),
    }
    p["ln1_g"], p["ln1_b"] = ln_params(h, f"{prefix}.ln1", layer)
    p["ln2_g"], p["ln2_b"] = ln_params(h, f"{prefix}.ln2", layer)
    return p


_NIBBLES_NO_M8 = np.array([0, 1, 2, 3, 4, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15], np.uint8)


def random_packed(rows: int, cols: int, name: str, full_range: bool = False) -> np.ndarray:
    """Random packed INT4 bytes [rows, cols/2]: two nibbles per byte drawn uniformly
    from [-7, 7] (two's complement), or from [-8, 7] with full_range=True."""
    g = rng(name)
    if full_range:
        return g.integers(0, 256, size=(rows, cols // 2), dtype=np.uint8)
    lo = _NIBBLES_NO_M8[g.integers(0, 15, size=(rows, cols // 2))]
    hi = _NIBBLES_NO_M8[g.integers(0, 15, size=(rows, cols // 2))]
    return (lo | (hi << 4)).astype(np.uint8)


def random_i8(rows: int, cols: int, name: str) -> np.ndarray:
    """Random int8 codes [rows, cols] uniform in [-127, 127] (W8A8 GEMM sweep operands)."""
    return rng(name).integers(-127, 128, size=(rows, cols), dtype=np.int8)


def random_scales(n: int, name: str) -> np.ndarray:
    return (rng(name).uniform(0.5, 1.5, n) / 16.0).astype(np.float32)
