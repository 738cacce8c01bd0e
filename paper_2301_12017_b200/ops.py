"""torch-facing wrappers over the C ABI (include/q4.h) -- marshalling only.

Tensors must be CUDA tensors of the documented dtype/shape; outputs are allocated with
torch and filled by the library on torch's current stream."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import (EPI_F16, EPI_GELU_Q4, EPI_I32, EPI_RESLN_Q4, Epilogue, LayerCfg,
                   LayerWeights, Taps, check, lib)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need(t, dtype, name, dims=None):
    if t is None:
        return
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dims is not None and t.dim() != dims:
        raise ValueError(f"{name} must be {dims}-D, got shape {tuple(t.shape)}")


def quantize_rows(x: torch.Tensor, clip: float = 0.0, codes=None, scales=None):
    """a1/a2: fp16 [rows, cols] -> (packed INT4 codes uint8 [rows, cols/2], fp32 scales [rows])."""
    _need(x, torch.float16, "x", 2)
    rows, cols = x.shape
    if codes is None:
        codes = torch.empty(rows, cols // 2, dtype=torch.uint8, device=x.device)
    if scales is None:
        scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    check(lib().q4_quantize_rows(_ptr(x), rows, cols, cols, clip, _ptr(codes), _ptr(scales), _stream()))
    return codes, scales


def w4a4_linear(a_codes, a_scales, w_codes, w_scales, kind=EPI_F16, *, bias=None, residual=None,
                gamma=None, beta=None, ln_eps=1e-12, clip=0.0, mainloop=0, f16_tap=False,
                out=None, workspace=None, w_i8=None, asym_out=False):
    """a3-a6: INT4 x INT4 -> exact INT32 -> fused epilogue.  Returns a dict with the
    outputs of the epilogue kind: i32 | f16 | (codes, scales[, zeros][, f16]).
    asym_out: the requantizing kinds write asymmetric codes + zeros (NEXT-3)."""
    _need(a_codes, torch.uint8, "a_codes", 2)
    _need(w_codes, torch.uint8, "w_codes", 2)
    _need(a_scales, torch.float32, "a_scales", 1)
    _need(w_scales, torch.float32, "w_scales", 1)
    for n, t in (("bias", bias), ("residual", residual), ("gamma", gamma), ("beta", beta)):
        _need(t, torch.float16, n)
    M, K = a_codes.shape[0], a_codes.shape[1] * 2
    N = w_codes.shape[0]
    if w_codes.shape[1] * 2 != K:
        raise ValueError(f"K mismatch: a_codes {tuple(a_codes.shape)} vs w_codes {tuple(w_codes.shape)}")
    dev = a_codes.device
    o = dict(out or {})
    if kind == EPI_I32:
        o.setdefault("i32", torch.empty(M, N, dtype=torch.int32, device=dev))
    if kind in (EPI_F16, EPI_RESLN_Q4) or (kind == EPI_GELU_Q4 and f16_tap):
        o.setdefault("f16", torch.empty(M, N, dtype=torch.float16, device=dev))
    if kind in (EPI_GELU_Q4, EPI_RESLN_Q4):
        o.setdefault("codes", torch.empty(M, N // 2, dtype=torch.uint8, device=dev))
        o.setdefault("scales", torch.empty(M, dtype=torch.float32, device=dev))
        if asym_out:
            o.setdefault("zeros", torch.empty(M, dtype=torch.float32, device=dev))
    e = Epilogue(kind=kind, mainloop=mainloop, bias=_ptr(bias), residual=_ptr(residual),
                 gamma=_ptr(gamma), beta=_ptr(beta), ln_eps=ln_eps, requant_clip=clip,
                 out_i32=_ptr(o.get("i32")), out_f16=_ptr(o.get("f16")),
                 out_codes=_ptr(o.get("codes")), out_scales=_ptr(o.get("scales")), w_i8=_ptr(w_i8),
                 out_zeros=_ptr(o.get("zeros")))
    ws_bytes = lib().q4_w4a4_linear_workspace(M, N, K, kind)
    if ws_bytes and workspace is None:  # a caller's workspace goes to the C ABI as given
        workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    check(lib().q4_w4a4_linear(_ptr(a_codes), _ptr(a_scales), _ptr(w_codes), _ptr(w_scales),
                               M, N, K, C.byref(e), _ptr(workspace),
                               0 if workspace is None else workspace.numel(), _stream()))
    return o


def quantize_rows_i8(x: torch.Tensor, clip: float = 0.0, codes=None, scales=None):
    """W8A8 baseline: fp16 [rows, cols] -> (int8 codes [rows, cols], fp32 scales = amax/127)."""
    _need(x, torch.float16, "x", 2)
    rows, cols = x.shape
    if codes is None:
        codes = torch.empty(rows, cols, dtype=torch.int8, device=x.device)
    if scales is None:
        scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    check(lib().q4_quantize_rows_i8(_ptr(x), rows, cols, cols, clip, _ptr(codes), _ptr(scales), _stream()))
    return codes, scales


def w8a8_linear(a_codes, a_scales, w_codes, w_scales, kind=EPI_F16, *, bias=None, residual=None,
                gamma=None, beta=None, ln_eps=1e-12, clip=0.0, f16_tap=False, out=None, workspace=None):
    """W8A8 baseline of w4a4_linear: int8 x int8 -> exact INT32 -> the same fused epilogues;
    requantizing kinds return int8 codes [M, N]."""
    _need(a_codes, torch.int8, "a_codes", 2)
    _need(w_codes, torch.int8, "w_codes", 2)
    _need(a_scales, torch.float32, "a_scales", 1)
    _need(w_scales, torch.float32, "w_scales", 1)
    for n, t in (("bias", bias), ("residual", residual), ("gamma", gamma), ("beta", beta)):
        _need(t, torch.float16, n)
    M, K = a_codes.shape
    N = w_codes.shape[0]
    if w_codes.shape[1] != K:
        raise ValueError(f"K mismatch: a_codes {tuple(a_codes.shape)} vs w_codes {tuple(w_codes.shape)}")
    dev = a_codes.device
    o = dict(out or {})
    if kind == EPI_I32:
        o.setdefault("i32", torch.empty(M, N, dtype=torch.int32, device=dev))
    if kind in (EPI_F16, EPI_RESLN_Q4) or (kind == EPI_GELU_Q4 and f16_tap):
        o.setdefault("f16", torch.empty(M, N, dtype=torch.float16, device=dev))
    if kind in (EPI_GELU_Q4, EPI_RESLN_Q4):
        o.setdefault("codes", torch.empty(M, N, dtype=torch.int8, device=dev))
        o.setdefault("scales", torch.empty(M, dtype=torch.float32, device=dev))
    e = Epilogue(kind=kind, mainloop=0, bias=_ptr(bias), residual=_ptr(residual),
                 gamma=_ptr(gamma), beta=_ptr(beta), ln_eps=ln_eps, requant_clip=clip,
                 out_i32=_ptr(o.get("i32")), out_f16=_ptr(o.get("f16")),
                 out_codes=_ptr(o.get("codes")), out_scales=_ptr(o.get("scales")), w_i8=None)
    ws_bytes = lib().q4_w8a8_linear_workspace(M, N, K, kind)
    if ws_bytes and workspace is None:  # a caller's workspace goes to the C ABI as given
        workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    check(lib().q4_w8a8_linear(_ptr(a_codes), _ptr(a_scales), _ptr(w_codes), _ptr(w_scales),
                               M, N, K, C.byref(e), _ptr(workspace),
                               0 if workspace is None else workspace.numel(), _stream()))
    return o


def f16_linear(a, w, kind=EPI_F16, *, bias=None, residual=None, gamma=None, beta=None, ln_eps=1e-12,
               clip=0.0, f16_tap=False, out=None, workspace=None):
    """FP16 linear (unquantized part of a per-part strategy): fp16 [M,K] x fp16 [N,K] on the
    tensor cores + the same fused epilogues (F16 | GELU_Q4 | RESLN_Q4, INT4 codes)."""
    _need(a, torch.float16, "a", 2)
    _need(w, torch.float16, "w", 2)
    for n, t in (("bias", bias), ("residual", residual), ("gamma", gamma), ("beta", beta)):
        _need(t, torch.float16, n)
    M, K = a.shape
    N = w.shape[0]
    if w.shape[1] != K:
        raise ValueError(f"K mismatch: a {tuple(a.shape)} vs w {tuple(w.shape)}")
    dev = a.device
    o = dict(out or {})
    if kind in (EPI_F16, EPI_RESLN_Q4) or (kind == EPI_GELU_Q4 and f16_tap):
        o.setdefault("f16", torch.empty(M, N, dtype=torch.float16, device=dev))
    if kind in (EPI_GELU_Q4, EPI_RESLN_Q4):
        o.setdefault("codes", torch.empty(M, N // 2, dtype=torch.uint8, device=dev))
        o.setdefault("scales", torch.empty(M, dtype=torch.float32, device=dev))
    e = Epilogue(kind=kind, mainloop=0, bias=_ptr(bias), residual=_ptr(residual),
                 gamma=_ptr(gamma), beta=_ptr(beta), ln_eps=ln_eps, requant_clip=clip,
                 out_i32=None, out_f16=_ptr(o.get("f16")),
                 out_codes=_ptr(o.get("codes")), out_scales=_ptr(o.get("scales")), w_i8=None)
    ws_bytes = lib().q4_f16_linear_workspace(M, N, K, kind)
    if ws_bytes and workspace is None:  # a caller's workspace goes to the C ABI as given
        workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    check(lib().q4_f16_linear(_ptr(a), _ptr(w), M, N, K, C.byref(e), _ptr(workspace),
                              0 if workspace is None else workspace.numel(), _stream()))
    return o


def quantize_rows_asym(x: torch.Tensor):
    """NEXT-3: fp16 [rows, cols] -> (unsigned INT4 codes uint8 [rows, cols/2], scales, zeros)."""
    _need(x, torch.float16, "x", 2)
    rows, cols = x.shape
    codes = torch.empty(rows, cols // 2, dtype=torch.uint8, device=x.device)
    scales = torch.empty(rows, dtype=torch.float32, device=x.device)
    zeros = torch.empty(rows, dtype=torch.float32, device=x.device)
    check(lib().q4_quantize_rows_asym(_ptr(x), rows, cols, cols, _ptr(codes), _ptr(scales), _ptr(zeros), _stream()))
    return codes, scales, zeros


def weight_code_sums(w_codes: torch.Tensor) -> torch.Tensor:
    _need(w_codes, torch.uint8, "w_codes", 2)
    N, K = w_codes.shape[0], w_codes.shape[1] * 2
    out = torch.empty(N, dtype=torch.float32, device=w_codes.device)
    check(lib().q4_weight_code_sums(_ptr(w_codes), N, K, _ptr(out), _stream()))
    return out


def w4a4_asym_linear(a_codes, a_scales, a_zeros, w_codes, w_scales, w_sums, kind=EPI_F16, *, bias=None,
                     residual=None, gamma=None, beta=None, ln_eps=1e-12, mainloop=0, w_i8=None, out=None,
                     f16_tap=False, asym_out=True, workspace=None):
    """NEXT-3: asymmetric activations x symmetric INT4 weights with the four epilogues; the
    requantizing kinds write asymmetric codes + zeros (asym_out) or symmetric codes."""
    _need(a_codes, torch.uint8, "a_codes", 2)
    _need(w_codes, torch.uint8, "w_codes", 2)
    M, K = a_codes.shape[0], a_codes.shape[1] * 2
    N = w_codes.shape[0]
    dev = a_codes.device
    o = dict(out or {})
    if kind == EPI_I32:
        o.setdefault("i32", torch.empty(M, N, dtype=torch.int32, device=dev))
    if kind in (EPI_F16, EPI_RESLN_Q4) or (kind == EPI_GELU_Q4 and f16_tap):
        o.setdefault("f16", torch.empty(M, N, dtype=torch.float16, device=dev))
    if kind in (EPI_GELU_Q4, EPI_RESLN_Q4):
        o.setdefault("codes", torch.empty(M, N // 2, dtype=torch.uint8, device=dev))
        o.setdefault("scales", torch.empty(M, dtype=torch.float32, device=dev))
        if asym_out:
            o.setdefault("zeros", torch.empty(M, dtype=torch.float32, device=dev))
    e = Epilogue(kind=kind, mainloop=mainloop, bias=_ptr(bias), residual=_ptr(residual), gamma=_ptr(gamma),
                 beta=_ptr(beta), ln_eps=ln_eps, requant_clip=0.0, out_i32=_ptr(o.get("i32")),
                 out_f16=_ptr(o.get("f16")), out_codes=_ptr(o.get("codes")), out_scales=_ptr(o.get("scales")),
                 w_i8=_ptr(w_i8), out_zeros=_ptr(o.get("zeros")))
    ws_bytes = lib().q4_w4a4_linear_workspace(M, N, K, kind)
    if ws_bytes and workspace is None:  # a caller's workspace goes to the C ABI as given
        workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    check(lib().q4_w4a4_asym_linear(_ptr(a_codes), _ptr(a_scales), _ptr(a_zeros), _ptr(w_codes), _ptr(w_scales),
                                    _ptr(w_sums), M, N, K, C.byref(e), _ptr(workspace),
                                    0 if workspace is None else workspace.numel(), _stream()))
    return o


def attention_f16_q4_asym(qkv, B, S, heads, head_dim=64):
    """NEXT-3 a7: fp16 QKV -> (ctx codes, scales, zeros, ctx fp16) with asymmetric ctx codes."""
    _need(qkv, torch.float16, "qkv", 2)
    h = heads * head_dim
    dev = qkv.device
    codes = torch.empty(B * S, h // 2, dtype=torch.uint8, device=dev)
    scales = torch.empty(B * S, dtype=torch.float32, device=dev)
    zeros = torch.empty(B * S, dtype=torch.float32, device=dev)
    ctx = torch.empty(B * S, h, dtype=torch.float16, device=dev)
    check(lib().q4_attention_f16_q4_asym(_ptr(qkv), B, S, heads, head_dim, _ptr(ctx), _ptr(codes), _ptr(scales),
                                         _ptr(zeros), _stream()))
    return codes, scales, zeros, ctx


def attention_f16_q4(qkv, B, S, heads, head_dim=64, f16_tap=False):
    """a7: fp16 QKV [B*S, 3h] -> (ctx codes [B*S, h/2], ctx scales [B*S][, ctx fp16])."""
    _need(qkv, torch.float16, "qkv", 2)
    h = heads * head_dim
    dev = qkv.device
    codes = torch.empty(B * S, h // 2, dtype=torch.uint8, device=dev)
    scales = torch.empty(B * S, dtype=torch.float32, device=dev)
    ctx = torch.empty(B * S, h, dtype=torch.float16, device=dev)
    check(lib().q4_attention_f16_q4(_ptr(qkv), B, S, heads, head_dim, _ptr(ctx), _ptr(codes),
                                    _ptr(scales), _stream()))
    return (codes, scales, ctx) if f16_tap else (codes, scales)


def attention_f16_q8(qkv, B, S, heads, head_dim=64, f16_tap=False):
    """W8A8 baseline of a7: (ctx int8 codes [B*S, h], ctx scales = amax/127[, ctx fp16])."""
    _need(qkv, torch.float16, "qkv", 2)
    h = heads * head_dim
    dev = qkv.device
    codes = torch.empty(B * S, h, dtype=torch.int8, device=dev)
    scales = torch.empty(B * S, dtype=torch.float32, device=dev)
    ctx = torch.empty(B * S, h, dtype=torch.float16, device=dev)
    check(lib().q4_attention_f16_q8(_ptr(qkv), B, S, heads, head_dim, _ptr(ctx), _ptr(codes),
                                    _ptr(scales), _stream()))
    return (codes, scales, ctx) if f16_tap else (codes, scales)


def layer_cfg(cfg: dict) -> LayerCfg:
    return LayerCfg(cfg["hidden"], cfg["heads"], cfg["head_dim"], cfg["ffn"], cfg.get("ln_eps", 1e-12),
                    int(cfg.get("fp16_parts", 0)), int(cfg.get("asym_acts", 0)))


def prune_24(w: torch.Tensor) -> torch.Tensor:
    """NEXT-4 offline: l1 Pair-(2:4) pruning of fp16 [N, K] weight rows (q4_prune_24)."""
    _need(w, torch.float16, "w", 2)
    out = torch.empty_like(w)
    check(lib().q4_prune_24(_ptr(w), w.shape[0], w.shape[1], _ptr(out), _stream()))
    return out


def sparse24_compress(w_codes: torch.Tensor):
    """NEXT-4 offline: packed 2:4-sparse INT4 codes -> (values int8 [N, K/2], metadata int32
    [N, K/32], violations) (q4_sparse24_compress)."""
    _need(w_codes, torch.uint8, "w_codes", 2)
    N, K = w_codes.shape[0], w_codes.shape[1] * 2
    vals = torch.empty(N, K // 2, dtype=torch.int8, device=w_codes.device)
    meta = torch.empty(N, K // 32, dtype=torch.int32, device=w_codes.device)
    bad = torch.zeros(1, dtype=torch.int32, device=w_codes.device)
    check(lib().q4_sparse24_compress(_ptr(w_codes), N, K, _ptr(vals), _ptr(meta), _ptr(bad), _stream()))
    return vals, meta, bad


def w4a4_sparse24_linear(a_codes, a_scales, w_vals, w_meta, w_scales, kind=EPI_F16, *, bias=None, out=None):
    """NEXT-4: INT4 activations x 2:4-sparse INT4 weights (compressed), F16 or I32 epilogue."""
    _need(a_codes, torch.uint8, "a_codes", 2)
    M, K = a_codes.shape[0], a_codes.shape[1] * 2
    N = w_vals.shape[0]
    o = dict(out or {})
    key = "i32" if kind == EPI_I32 else "f16"
    o.setdefault(key, torch.empty(M, N, dtype=torch.int32 if kind == EPI_I32 else torch.float16, device=a_codes.device))
    e = Epilogue(kind=kind, bias=_ptr(bias), out_i32=_ptr(o.get("i32")), out_f16=_ptr(o.get("f16")))
    check(lib().q4_w4a4_sparse24_linear(_ptr(a_codes), _ptr(a_scales), _ptr(w_vals), _ptr(w_meta), _ptr(w_scales),
                                        M, N, K, C.byref(e), _stream()))
    return o


def launch_floor(n: int, ctas: int = 32):
    """Measurement only: n empty PDL kernels on the current stream (q4_launch_floor)."""
    _lib.check(_lib.lib().q4_launch_floor(int(n), int(ctas), _stream()), "q4_launch_floor")


def prepack_weights(w_codes: torch.Tensor) -> torch.Tensor:
    """a2': packed INT4 [N, K/2] -> MMA-ready int8 [N, K] (q4_prepack_weights)."""
    _need(w_codes, torch.uint8, "w_codes", 2)
    N, K = w_codes.shape[0], w_codes.shape[1] * 2
    out = torch.empty(N, K, dtype=torch.int8, device=w_codes.device)
    check(lib().q4_prepack_weights(_ptr(w_codes), N, K, _ptr(out), _stream()))
    return out


def layer_weights(w: dict) -> LayerWeights:
    """w: dict of CUDA tensors (codes uint8, scales fp32, biases / LN params fp16; the
    optional prepacked int8 copies wqkv8 / wo8 / w18 / w28)."""
    return LayerWeights(**{k: (w[k].data_ptr() if w.get(k) is not None else None)
                           for k in _lib.WEIGHT_FIELDS})


def quantize_layer(params: dict, device="cuda", prepack: bool = True, bits: int = 4,
                   fp16_parts: int = 0, asym: bool = False) -> dict:
    """Offline weight prep (a2, not timed): fp16 [out, in] weights -> per-output-channel
    INT4 codes + scales on the device (and, with prepack, the MMA-ready int8 copy);
    biases and LN parameters copied as fp16.  bits=8: the W8A8 baseline's int8 codes.
    fp16_parts (strategy bits, q4_layer_cfg): those parts also keep their fp16 weights
    (fqkv / fo / f1 / f2)."""
    if bits not in (4, 8):
        raise ValueError(f"bits={bits} (4 or 8)")
    w = {}
    for i, k in enumerate(("wqkv", "wo", "w1", "w2")):
        t = torch.as_tensor(params[k]).to(device=device, dtype=torch.float16).contiguous()
        if fp16_parts >> i & 1:
            w["f" + k[1:]] = t
        if bits == 8:
            w[k], w["s" + k[1:]] = quantize_rows_i8(t)
            continue
        w[k], w["s" + k[1:]] = quantize_rows(t)
        if prepack:
            w[k + "8"] = prepack_weights(w[k])
        if asym:  # asymmetric activations: the zero-point term's weight code sums (NEXT-3)
            w["c" + k[1:]] = weight_code_sums(w[k])
    for k in ("bqkv", "bo", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"):
        w[k] = torch.as_tensor(params[k]).to(device=device, dtype=torch.float16).contiguous()
    return w


def encoder_layer_workspace_bytes(cfg: dict, B: int, S: int, bits: int = 4) -> int:
    """q4_encoder_layer_workspace (bits=8: the W8A8 layer's)."""
    lc = layer_cfg(cfg)
    fn = lib().q4_encoder_layer_w8a8_workspace if bits == 8 else lib().q4_encoder_layer_workspace
    return int(fn(C.byref(lc), B, S))


def encoder_layer(cfg: dict, w: dict, B: int, S: int, h_in, hq_in, hs_in, taps: bool = False,
                  workspace=None, bits: int = 4, hz_in=None):
    """a8: one post-LN BERT layer (qall).  Returns dict(h_out, hq_out, hs_out[, taps...]).
    bits=8: the W8A8 baseline (q4_encoder_layer_w8a8; int8 codes, weights from
    quantize_layer(bits=8))."""
    M, h, f = B * S, cfg["hidden"], cfg["ffn"]
    dev = h_in.device
    lc = layer_cfg(cfg)
    i8 = bits == 8
    ws_bytes = (lib().q4_encoder_layer_w8a8_workspace if i8 else lib().q4_encoder_layer_workspace)(C.byref(lc), B, S)
    if workspace is None:
        workspace = torch.zeros(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    cdt, cdiv = (torch.int8, 1) if i8 else (torch.uint8, 2)
    asym = bool(cfg.get("asym_acts", 0))
    out = {"h_out": torch.empty(M, h, dtype=torch.float16, device=dev),
           "hq_out": torch.empty(M, h // cdiv, dtype=cdt, device=dev),
           "hs_out": torch.empty(M, dtype=torch.float32, device=dev)}
    if asym:
        out["hz_out"] = torch.empty(M, dtype=torch.float32, device=dev)
    tp = None
    if taps:
        shapes = {"qkv": ((M, 3 * h), torch.float16), "ctx": ((M, h), torch.float16),
                  "h1": ((M, h), torch.float16), "ffn1": ((M, f), torch.float16),
                  "acc_qkv": ((M, 3 * h), torch.int32), "acc_o": ((M, h), torch.int32),
                  "acc_1": ((M, f), torch.int32), "acc_2": ((M, h), torch.int32),
                  "ctx_codes": ((M, h // cdiv), cdt), "h1_codes": ((M, h // cdiv), cdt),
                  "f_codes": ((M, f // cdiv), cdt), "ctx_scales": ((M,), torch.float32),
                  "h1_scales": ((M,), torch.float32), "f_scales": ((M,), torch.float32)}
        if asym:
            shapes.update({k: ((M,), torch.float32) for k in ("ctx_zeros", "h1_zeros", "f_zeros")})
        for k, (shp, dt) in shapes.items():
            out[k] = torch.empty(shp, dtype=dt, device=dev)
        tp = Taps(**{k: (out[k].data_ptr() if k in out else None) for k in _lib.TAP_FIELDS})
    lw = layer_weights(w)
    tpp = C.byref(tp) if tp is not None else None
    if asym:
        check(lib().q4_encoder_layer_asym(C.byref(lc), C.byref(lw), B, S, _ptr(h_in), _ptr(hq_in), _ptr(hs_in),
                                          _ptr(hz_in), _ptr(out["h_out"]), _ptr(out["hq_out"]), _ptr(out["hs_out"]),
                                          _ptr(out["hz_out"]), _ptr(workspace), workspace.numel(), tpp, _stream()))
        return out
    fn = lib().q4_encoder_layer_w8a8 if i8 else lib().q4_encoder_layer
    check(fn(C.byref(lc), C.byref(lw), B, S, _ptr(h_in), _ptr(hq_in),
                                 _ptr(hs_in), _ptr(out["h_out"]), _ptr(out["hq_out"]),
                                 _ptr(out["hs_out"]), _ptr(workspace), workspace.numel(),
                                 tpp, _stream()))
    return out
