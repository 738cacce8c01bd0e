"""ctypes binding of libq4.so (include/q4.h).  Argument marshalling only: every step of
the hot path runs in the CUDA kernels behind the C ABI.  torch supplies device memory
and the current stream.  There is no fallback: if the library is missing or a call
fails, this raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# Q4_LIB_PATH: profiling only (A/B timing of two builds); the default is the in-tree build
LIB_PATH = os.environ.get("Q4_LIB_PATH") or os.path.join(HERE, "libq4.so")

Q4_OK, Q4_EINVAL, Q4_ESHAPE, Q4_EALIGN, Q4_EUNSUPPORTED, Q4_ECUDA = range(6)
EPI_I32, EPI_F16, EPI_GELU_Q4, EPI_RESLN_Q4 = range(4)
(MAINLOOP_AUTO, MAINLOOP_TCGEN05, MAINLOOP_MMA_SYNC_S8, MAINLOOP_MMA_SYNC_S4, MAINLOOP_TCGEN05_W8,
 MAINLOOP_TCGEN05_W8_1CTA) = range(6)
STATUS_NAMES = ["Q4_OK", "Q4_EINVAL", "Q4_ESHAPE", "Q4_EALIGN", "Q4_EUNSUPPORTED", "Q4_ECUDA"]

EXPORTS = (
    "q4_last_error", "q4_version", "q4_launch_count", "q4_quantize_rows", "q4_prepack_weights",
    "q4_w4a4_linear_workspace", "q4_w4a4_linear", "q4_attention_f16_q4",
    "q4_encoder_layer_workspace", "q4_encoder_layer", "q4_encoder_stack_workspace",
    "q4_encoder_stack", "q4_quantize_rows_i8", "q4_w8a8_linear_workspace", "q4_w8a8_linear",
    "q4_attention_f16_q8", "q4_encoder_layer_w8a8_workspace", "q4_encoder_layer_w8a8",
    "q4_encoder_stack_w8a8_workspace", "q4_encoder_stack_w8a8", "q4_f16_linear_workspace", "q4_f16_linear",
    "q4_quantize_rows_asym", "q4_weight_code_sums", "q4_w4a4_asym_linear",
    "q4_encoder_pipeline_workspace", "q4_encoder_pipeline", "q4_launch_floor", "q4_attention_f16_q4_asym",
    "q4_encoder_layer_asym", "q4_prune_24", "q4_sparse24_compress", "q4_w4a4_sparse24_linear",
)


class Q4Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 6 else status}: {msg}")
        self.status = status


class Epilogue(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("mainloop", C.c_int32),
        ("bias", C.c_void_p), ("residual", C.c_void_p), ("gamma", C.c_void_p), ("beta", C.c_void_p),
        ("ln_eps", C.c_float), ("requant_clip", C.c_float),
        ("out_i32", C.c_void_p), ("out_f16", C.c_void_p), ("out_codes", C.c_void_p),
        ("out_scales", C.c_void_p), ("w_i8", C.c_void_p), ("out_zeros", C.c_void_p),
    ]


class LayerCfg(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("heads", C.c_int32), ("head_dim", C.c_int32),
                ("ffn", C.c_int32), ("ln_eps", C.c_float), ("fp16_parts", C.c_int32), ("asym_acts", C.c_int32)]


WEIGHT_FIELDS = ("wqkv", "wo", "w1", "w2", "wqkv8", "wo8", "w18", "w28", "sqkv", "so", "s1", "s2",
                 "bqkv", "bo", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b", "fqkv", "fo", "f1", "f2",
                 "cqkv", "co", "c1", "c2")
TAP_FIELDS = ("qkv", "ctx", "h1", "ffn1", "acc_qkv", "acc_o", "acc_1", "acc_2", "ctx_codes",
              "h1_codes", "f_codes", "ctx_scales", "h1_scales", "f_scales", "ctx_zeros", "h1_zeros", "f_zeros")


class LayerWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in WEIGHT_FIELDS]


class Taps(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in TAP_FIELDS]


_lib = None


def lib():
    """Load libq4.so (raises if it was not built -- there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: build it with "
                              f"`python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P, I64, I32, F, SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_size_t
        L.q4_last_error.restype = C.c_char_p
        L.q4_version.restype = C.c_char_p
        L.q4_launch_count.restype = C.c_uint64
        L.q4_quantize_rows.argtypes = [P, I64, I64, I64, F, P, P, P]
        L.q4_prepack_weights.argtypes = [P, I64, I64, P, P]
        L.q4_w4a4_linear_workspace.argtypes = [I64, I64, I64, I32]
        L.q4_w4a4_linear_workspace.restype = SZ
        L.q4_w4a4_linear.argtypes = [P, P, P, P, I64, I64, I64, C.POINTER(Epilogue), P, SZ, P]
        L.q4_attention_f16_q4.argtypes = [P, I64, I64, I32, I32, P, P, P, P]
        L.q4_quantize_rows_i8.argtypes = [P, I64, I64, I64, F, P, P, P]
        L.q4_w8a8_linear_workspace.argtypes = [I64, I64, I64, I32]
        L.q4_w8a8_linear_workspace.restype = SZ
        L.q4_w8a8_linear.argtypes = [P, P, P, P, I64, I64, I64, C.POINTER(Epilogue), P, SZ, P]
        L.q4_encoder_layer_workspace.argtypes = [C.POINTER(LayerCfg), I64, I64]
        L.q4_encoder_layer_workspace.restype = SZ
        L.q4_encoder_layer.argtypes = [C.POINTER(LayerCfg), C.POINTER(LayerWeights), I64, I64, P, P, P,
                                       P, P, P, P, SZ, C.POINTER(Taps), P]
        L.q4_encoder_stack_workspace.argtypes = [C.POINTER(LayerCfg), I64, I64]
        L.q4_encoder_stack_workspace.restype = SZ
        L.q4_encoder_stack.argtypes = [C.POINTER(LayerCfg), C.POINTER(LayerWeights), I32, I64, I64, P,
                                       P, P, SZ, P]
        L.q4_attention_f16_q8.argtypes = [P, I64, I64, I32, I32, P, P, P, P]
        L.q4_f16_linear_workspace.argtypes = [I64, I64, I64, I32]
        L.q4_f16_linear_workspace.restype = SZ
        L.q4_f16_linear.argtypes = [P, P, I64, I64, I64, C.POINTER(Epilogue), P, SZ, P]
        L.q4_quantize_rows_asym.argtypes = [P, I64, I64, I64, P, P, P, P]
        L.q4_encoder_pipeline_workspace.argtypes = [C.POINTER(LayerCfg), I64, I64]
        L.q4_encoder_pipeline_workspace.restype = SZ
        L.q4_encoder_pipeline.argtypes = [C.POINTER(LayerCfg), C.POINTER(LayerWeights), I32, I64, I64, P, P, I32,
                                          P, SZ, P]
        L.q4_weight_code_sums.argtypes = [P, I64, I64, P, P]
        L.q4_w4a4_asym_linear.argtypes = [P, P, P, P, P, P, I64, I64, I64, C.POINTER(Epilogue), P, SZ, P]
        L.q4_prune_24.argtypes = [P, I64, I64, P, P]
        L.q4_sparse24_compress.argtypes = [P, I64, I64, P, P, P, P]
        L.q4_w4a4_sparse24_linear.argtypes = [P, P, P, P, P, I64, I64, I64, C.POINTER(Epilogue), P]
        L.q4_attention_f16_q4_asym.argtypes = [P, I64, I64, I32, I32, P, P, P, P, P]
        L.q4_encoder_layer_asym.argtypes = [C.POINTER(LayerCfg), C.POINTER(LayerWeights), I64, I64, P, P, P, P,
                                            P, P, P, P, P, SZ, C.POINTER(Taps), P]
        L.q4_encoder_layer_w8a8_workspace.argtypes = [C.POINTER(LayerCfg), I64, I64]
        L.q4_encoder_layer_w8a8_workspace.restype = SZ
        L.q4_encoder_layer_w8a8.argtypes = L.q4_encoder_layer.argtypes
        L.q4_encoder_stack_w8a8_workspace.argtypes = [C.POINTER(LayerCfg), I64, I64]
        L.q4_encoder_stack_w8a8_workspace.restype = SZ
        L.q4_encoder_stack_w8a8.argtypes = L.q4_encoder_stack.argtypes
        L.q4_launch_floor.argtypes = [C.c_int32, C.c_int32, P]
        for name in EXPORTS:
            L[name].restype = L[name].restype if name in (
                "q4_last_error", "q4_version", "q4_launch_count", "q4_w4a4_linear_workspace",
                "q4_encoder_layer_workspace", "q4_encoder_stack_workspace",
                "q4_w8a8_linear_workspace", "q4_encoder_layer_w8a8_workspace",
                "q4_encoder_stack_w8a8_workspace", "q4_f16_linear_workspace",
                "q4_encoder_pipeline_workspace") else C.c_int
        _lib = L
    return _lib


def check(status: int, what: str = ""):
    if status != Q4_OK:
        raise Q4Error(status, (lib().q4_last_error() or b"").decode() or what)


def version() -> str:
    return lib().q4_version().decode()


def launch_count() -> int:
    return int(lib().q4_launch_count())
