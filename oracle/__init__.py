"""CPU oracle for the W4A4 encoder hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2301_12017_b200``) never imports it and shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around ``oracle.c``; the
arithmetic, with its citations of PAPER.md, lives there.  fp16 tensors cross the
boundary as ``np.float16`` arrays (their bit patterns are passed as uint16).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

EPI_I32, EPI_F16, EPI_GELU_Q4, EPI_RESLN_Q4 = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain C11, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = [
            "gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-fopenmp",
            "-ffp-contract=off", "-fno-fast-math", "-Wall", "-Wno-unknown-pragmas",
            _SRC, "-o", tmp, "-lm",
        ]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P, I64, I, F, D = C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_double
        L.oracle_f16_to_f64.argtypes = [C.c_uint16]
        L.oracle_f16_to_f64.restype = D
        L.oracle_f64_to_f16.argtypes = [D]
        L.oracle_f64_to_f16.restype = C.c_uint16
        L.oracle_quantize_rows.argtypes = [P, I64, I64, I64, F, P, P, I]
        L.oracle_pack_int4.argtypes = [P, I64, I64, P, P]
        L.oracle_unpack_int4.argtypes = [P, I64, I64, P]
        L.oracle_unpack_int4.restype = None
        L.oracle_gemm_i32.argtypes = [P, P, I64, I64, I64, P, I]
        L.oracle_w4a4_linear.argtypes = [P, P, P, P, I64, I64, I64, I, P, P, P, P, D, F,
                                         P, P, P, P, I]
        L.oracle_attention.argtypes = [P, I64, I64, I, I, P, P, P, I]
        L.oracle_encoder_layer.argtypes = [P, P, I64, I64, P, P, P, P, P, P, P, I]
        L.oracle_quantize_rows_i8.argtypes = [P, I64, I64, I64, F, P, P, I]
        L.oracle_gemm_i32_i8.argtypes = [P, P, I64, I64, I64, P, I]
        L.oracle_w8a8_linear.argtypes = [P, P, P, P, I64, I64, I64, I, P, P, P, P, D, F,
                                         P, P, P, P, I]
        L.oracle_f16_linear.argtypes = [P, P, I64, I64, I64, I, P, P, P, P, D, F, P, P, P, I]
        L.oracle_quantize_rows_asym.argtypes = [P, I64, I64, I64, P, P, P, I]
        L.oracle_prune_24.argtypes = [P, I64, I64, P]
        L.oracle_w4a4_asym_linear.argtypes = [P, P, P, P, P, I64, I64, I64, I, P, P, P, P, D, P, P, P, P, P, I]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed (rc={rc})")


# ---------------------------------------------------------------- fp16 helpers
def f16_to_f64(bits: int) -> float:
    return lib().oracle_f16_to_f64(int(bits))


def f64_to_f16_bits(v: float) -> int:
    return int(lib().oracle_f64_to_f16(float(v)))


# ---------------------------------------------------------------- O-1 / O-2
def quantize_rows(x: np.ndarray, clip: float = 0.0, threads: int = 0):
    """O-1: x fp16 [rows, cols] -> (codes uint8 [rows, ceil(cols/2)], scales fp32 [rows])."""
    x = _c(x, np.float16)
    rows, cols = x.shape
    codes = np.zeros((rows, (cols + 1) // 2), np.uint8)
    scales = np.zeros(rows, np.float32)
    _check(lib().oracle_quantize_rows(_p(x), rows, cols, cols, clip, _p(codes), _p(scales),
                                      threads), "quantize_rows")
    return codes, scales


def pack_int4(q: np.ndarray) -> np.ndarray:
    q = _c(q, np.int8)
    rows, cols = q.shape
    out = np.zeros((rows, (cols + 1) // 2), np.uint8)
    bad = C.c_int64(-1)
    rc = lib().oracle_pack_int4(_p(q), rows, cols, _p(out), C.byref(bad))
    if rc != 0:
        r, c = divmod(bad.value, cols)
        raise ValueError(f"pack_int4: value {int(q.flat[bad.value])} at ({r}, {c}) "
                         f"outside [-8, 7]")
    return out


def unpack_int4(packed: np.ndarray, cols: int) -> np.ndarray:
    packed = _c(packed, np.uint8)
    rows = packed.shape[0]
    q = np.zeros((rows, cols), np.int8)
    lib().oracle_unpack_int4(_p(packed), rows, cols, _p(q))
    return q


# ---------------------------------------------------------------- O-4 .. O-7
def gemm_i32(a_codes, w_codes, M, N, K, threads: int = 0) -> np.ndarray:
    a_codes, w_codes = _c(a_codes, np.uint8), _c(w_codes, np.uint8)
    acc = np.zeros((M, N), np.int32)
    _check(lib().oracle_gemm_i32(_p(a_codes), _p(w_codes), M, N, K, _p(acc), threads), "gemm")
    return acc


def w4a4_linear(a_codes, a_scales, w_codes, w_scales, M, N, K, epi=EPI_F16, bias=None,
                residual=None, gamma=None, beta=None, ln_eps=1e-12, clip=0.0,
                want_f16=True, threads: int = 0):
    """O-5..O-7.  Returns dict with keys among i32, f16, codes, scales."""
    a_codes, w_codes = _c(a_codes, np.uint8), _c(w_codes, np.uint8)
    a_scales, w_scales = _c(a_scales, np.float32), _c(w_scales, np.float32)
    bias, residual = _c(bias, np.float16), _c(residual, np.float16)
    gamma, beta = _c(gamma, np.float16), _c(beta, np.float16)
    out = {}
    i32 = f16 = codes = scales = None
    if epi == EPI_I32:
        i32 = out["i32"] = np.zeros((M, N), np.int32)
    if epi == EPI_F16 or epi == EPI_RESLN_Q4 or (epi == EPI_GELU_Q4 and want_f16):
        f16 = out["f16"] = np.zeros((M, N), np.float16)
    if epi in (EPI_GELU_Q4, EPI_RESLN_Q4):
        codes = out["codes"] = np.zeros((M, (N + 1) // 2), np.uint8)
        scales = out["scales"] = np.zeros(M, np.float32)
    rc = lib().oracle_w4a4_linear(_p(a_codes), _p(a_scales), _p(w_codes), _p(w_scales), M, N, K,
                                  epi, _p(bias), _p(residual), _p(gamma), _p(beta), ln_eps, clip,
                                  _p(i32), _p(f16), _p(codes), _p(scales), threads)
    _check(rc, "w4a4_linear")
    return out


# ---------------------------------------------------------------- O-11 .. O-13 (W8A8)
def quantize_rows_i8(x: np.ndarray, clip: float = 0.0, threads: int = 0):
    """O-11: x fp16 [rows, cols] -> (codes int8 [rows, cols], scales fp32 [rows] = fl32(amax/127))."""
    x = _c(x, np.float16)
    rows, cols = x.shape
    codes = np.zeros((rows, cols), np.int8)
    scales = np.zeros(rows, np.float32)
    _check(lib().oracle_quantize_rows_i8(_p(x), rows, cols, cols, clip, _p(codes), _p(scales),
                                         threads), "quantize_rows_i8")
    return codes, scales


def gemm_i32_i8(a_codes, w_codes, M, N, K, threads: int = 0) -> np.ndarray:
    """O-12: exact int8 x int8 GEMM, acc [M, N] int32."""
    a_codes, w_codes = _c(a_codes, np.int8), _c(w_codes, np.int8)
    acc = np.zeros((M, N), np.int32)
    _check(lib().oracle_gemm_i32_i8(_p(a_codes), _p(w_codes), M, N, K, _p(acc), threads), "gemm_i8")
    return acc


def w8a8_linear(a_codes, a_scales, w_codes, w_scales, M, N, K, epi=EPI_F16, bias=None,
                residual=None, gamma=None, beta=None, ln_eps=1e-12, clip=0.0,
                want_f16=True, threads: int = 0):
    """O-13: the W4A4 epilogues on the int8 accumulator; requant kinds give int8 codes."""
    a_codes, w_codes = _c(a_codes, np.int8), _c(w_codes, np.int8)
    a_scales, w_scales = _c(a_scales, np.float32), _c(w_scales, np.float32)
    bias, residual = _c(bias, np.float16), _c(residual, np.float16)
    gamma, beta = _c(gamma, np.float16), _c(beta, np.float16)
    out = {}
    i32 = f16 = codes = scales = None
    if epi == EPI_I32:
        i32 = out["i32"] = np.zeros((M, N), np.int32)
    if epi == EPI_F16 or epi == EPI_RESLN_Q4 or (epi == EPI_GELU_Q4 and want_f16):
        f16 = out["f16"] = np.zeros((M, N), np.float16)
    if epi in (EPI_GELU_Q4, EPI_RESLN_Q4):
        codes = out["codes"] = np.zeros((M, N), np.int8)
        scales = out["scales"] = np.zeros(M, np.float32)
    rc = lib().oracle_w8a8_linear(_p(a_codes), _p(a_scales), _p(w_codes), _p(w_scales), M, N, K,
                                  epi, _p(bias), _p(residual), _p(gamma), _p(beta), ln_eps, clip,
                                  _p(i32), _p(f16), _p(codes), _p(scales), threads)
    _check(rc, "w8a8_linear")
    return out


def f16_linear(a, w, M, N, K, epi=EPI_F16, bias=None, residual=None, gamma=None, beta=None,
               ln_eps=1e-12, clip=0.0, want_f16=True, threads: int = 0):
    """O-14: fp16 operands, fp64 sum, the O-5..O-7 epilogues (INT4 codes for *_Q4)."""
    a, w = _c(a, np.float16), _c(w, np.float16)
    bias, residual = _c(bias, np.float16), _c(residual, np.float16)
    gamma, beta = _c(gamma, np.float16), _c(beta, np.float16)
    out = {}
    f16 = codes = scales = None
    if epi == EPI_F16 or epi == EPI_RESLN_Q4 or (epi == EPI_GELU_Q4 and want_f16):
        f16 = out["f16"] = np.zeros((M, N), np.float16)
    if epi in (EPI_GELU_Q4, EPI_RESLN_Q4):
        codes = out["codes"] = np.zeros((M, (N + 1) // 2), np.uint8)
        scales = out["scales"] = np.zeros(M, np.float32)
    rc = lib().oracle_f16_linear(_p(a), _p(w), M, N, K, epi, _p(bias), _p(residual), _p(gamma), _p(beta),
                                 ln_eps, clip, _p(f16), _p(codes), _p(scales), threads)
    _check(rc, "f16_linear")
    return out


# ---------------------------------------------------------------- O-15 / O-16 (asymmetric)
def quantize_rows_asym(x: np.ndarray, threads: int = 0):
    """O-15: x fp16 [rows, cols] -> (codes uint8 [rows, cols/2] unsigned nibbles, scales, zeros)."""
    x = _c(x, np.float16)
    rows, cols = x.shape
    codes = np.zeros((rows, (cols + 1) // 2), np.uint8)
    scales = np.zeros(rows, np.float32)
    zeros = np.zeros(rows, np.float32)
    _check(lib().oracle_quantize_rows_asym(_p(x), rows, cols, cols, _p(codes), _p(scales), _p(zeros), threads),
           "quantize_rows_asym")
    return codes, scales, zeros


def unpack_u4(packed: np.ndarray, cols: int) -> np.ndarray:
    """Unsigned nibbles (low = even index) -> uint8 [rows, cols] in [0, 15]."""
    packed = np.asarray(packed, np.uint8)
    q = np.zeros((packed.shape[0], cols), np.uint8)
    q[:, 0::2] = packed[:, : (cols + 1) // 2] & 0xF
    q[:, 1::2] = packed[:, : cols // 2] >> 4
    return q


def w4a4_asym_linear(a_codes, a_scales, a_zeros, w_codes, w_scales, M, N, K, epi=EPI_F16, bias=None,
                     residual=None, gamma=None, beta=None, ln_eps=1e-12, asym_out=True, threads: int = 0):
    """O-16: asymmetric-activation W4A4 linear with the O-4..O-7 epilogues; the requantizing
    kinds code their fp16 output asymmetrically (O-15: codes, scales, zeros) when asym_out,
    else symmetrically (O-1: codes, scales)."""
    a_codes, w_codes = _c(a_codes, np.uint8), _c(w_codes, np.uint8)
    a_scales, a_zeros, w_scales = _c(a_scales, np.float32), _c(a_zeros, np.float32), _c(w_scales, np.float32)
    bias, residual = _c(bias, np.float16), _c(residual, np.float16)
    gamma, beta = _c(gamma, np.float16), _c(beta, np.float16)
    out = {}
    i32 = f16 = codes = scales = zeros = None
    if epi == EPI_I32:
        i32 = out["i32"] = np.zeros((M, N), np.int32)
    else:
        f16 = out["f16"] = np.zeros((M, N), np.float16)
    if epi in (EPI_GELU_Q4, EPI_RESLN_Q4):
        codes = out["codes"] = np.zeros((M, (N + 1) // 2), np.uint8)
        scales = out["scales"] = np.zeros(M, np.float32)
        if asym_out:
            zeros = out["zeros"] = np.zeros(M, np.float32)
    rc = lib().oracle_w4a4_asym_linear(_p(a_codes), _p(a_scales), _p(a_zeros), _p(w_codes), _p(w_scales), M, N, K,
                                       epi, _p(bias), _p(residual), _p(gamma), _p(beta), float(ln_eps), _p(i32),
                                       _p(f16), _p(codes), _p(scales), _p(zeros), threads)
    _check(rc, "w4a4_asym_linear")
    return out


# ---------------------------------------------------------------- O-17 (2:4 pruning)
def prune_24(w: np.ndarray) -> np.ndarray:
    """O-17: l1 Pair-(2:4) pruning of fp16 rows along K."""
    w = _c(w, np.float16)
    N, K = w.shape
    out = np.zeros_like(w)
    _check(lib().oracle_prune_24(_p(w.view(np.uint16)), N, K, _p(out.view(np.uint16))), "prune_24")
    return out


def attention(qkv, B, S, heads, head_dim, threads: int = 0):
    """O-8: returns (ctx fp16 [B*S, h], codes, scales)."""
    qkv = _c(qkv, np.float16)
    h = heads * head_dim
    ctx = np.zeros((B * S, h), np.float16)
    codes = np.zeros((B * S, h // 2), np.uint8)
    scales = np.zeros(B * S, np.float32)
    _check(lib().oracle_attention(_p(qkv), B, S, heads, head_dim, _p(ctx), _p(codes),
                                  _p(scales), threads), "attention")
    return ctx, codes, scales


class _Cfg(C.Structure):
    _fields_ = [("hidden", C.c_int), ("heads", C.c_int), ("head_dim", C.c_int),
                ("ffn", C.c_int), ("ln_eps", C.c_double)]


class _W(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "wqkv", "wo", "w1", "w2", "sqkv", "so", "s1", "s2",
        "bqkv", "bo", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")]


class _Taps(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "qkv", "ctx", "h1", "ffn1", "ctx_codes", "h1_codes", "f_codes",
        "ctx_scales", "h1_scales", "f_scales")]


def encoder_layer(cfg: dict, w: dict, B: int, S: int, h_in, hq_in, hs_in, taps: bool = False,
                  threads: int = 0):
    """O-9.  w holds quantized weights: wqkv/wo/w1/w2 (uint8 packed), sqkv/so/s1/s2
    (fp32), bqkv/bo/b1/b2/ln1_g/ln1_b/ln2_g/ln2_b (fp16).  Returns dict of outputs
    (h_out, hq_out, hs_out and, with taps=True, every intermediate)."""
    h, f = cfg["hidden"], cfg["ffn"]
    M = B * S
    keep = []

    def arr(a, dt):
        a = _c(a, dt)
        keep.append(a)
        return a

    W = _W(**{k: arr(w[k], np.uint8).ctypes.data for k in ("wqkv", "wo", "w1", "w2")},
           **{k: arr(w[k], np.float32).ctypes.data for k in ("sqkv", "so", "s1", "s2")},
           **{k: arr(w[k], np.float16).ctypes.data for k in (
               "bqkv", "bo", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")})
    cf = _Cfg(h, cfg["heads"], cfg["head_dim"], f, cfg.get("ln_eps", 1e-12))
    out = {"h_out": np.zeros((M, h), np.float16), "hq_out": np.zeros((M, h // 2), np.uint8),
           "hs_out": np.zeros(M, np.float32)}
    tp = None
    if taps:
        shapes = {"qkv": ((M, 3 * h), np.float16), "ctx": ((M, h), np.float16),
                  "h1": ((M, h), np.float16), "ffn1": ((M, f), np.float16),
                  "ctx_codes": ((M, h // 2), np.uint8), "h1_codes": ((M, h // 2), np.uint8),
                  "f_codes": ((M, f // 2), np.uint8), "ctx_scales": ((M,), np.float32),
                  "h1_scales": ((M,), np.float32), "f_scales": ((M,), np.float32)}
        for k, (shp, dt) in shapes.items():
            out[k] = np.zeros(shp, dt)
        tp = _Taps(**{k: out[k].ctypes.data for k in shapes})
    h_in, hq_in, hs_in = arr(h_in, np.float16), arr(hq_in, np.uint8), arr(hs_in, np.float32)
    rc = lib().oracle_encoder_layer(C.byref(cf), C.byref(W), B, S, _p(h_in), _p(hq_in),
                                    _p(hs_in), _p(out["h_out"]), _p(out["hq_out"]),
                                    _p(out["hs_out"]), C.byref(tp) if tp else None, threads)
    _check(rc, "encoder_layer")
    return out
