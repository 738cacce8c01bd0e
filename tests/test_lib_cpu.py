"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol
include/q4.h declares, and validates arguments synchronously (no compute calls)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2301_12017_b200 import build
    build.build()
    from paper_2301_12017_b200 import _lib
    return _lib.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "q4.h")).read()
    return sorted(set(re.findall(r"^Q4_API\s+[\w\s\*]+?\b(q4_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("q4_quantize_rows", "q4_w4a4_linear", "q4_attention_f16_q4", "q4_encoder_layer",
              "q4_encoder_stack", "q4_last_error"):
        assert s in syms
    from paper_2301_12017_b200 import _lib
    assert sorted(_lib.EXPORTS) == syms


def test_library_exports_every_declared_symbol(L):
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_version(L):
    assert b"sm_100a" in L.q4_version()


def test_shipped_library_has_no_profiling_knobs(L):
    """The profiling environment knobs (skip TMA / unpack / MMA / epilogue math, zero codes,
    trace stamps, tile / pair overrides) exist only in the -DQ4_PROFILING build: the shipped
    libq4.so does not even contain their names, so no stray variable can change its results."""
    from paper_2301_12017_b200 import _lib
    blob = open(_lib.LIB_PATH if not os.environ.get("Q4_LIB_PATH") else
                os.path.join(ROOT, "paper_2301_12017_b200", "libq4.so"), "rb").read()
    for k in (b"Q4_DEBUG_SKIP", b"Q4_TRACE", b"Q4_PAIR", b"Q4_TN", b"Q4_NO_PDL", b"Q4_ATTN_DBG",
              b"Q4_ATTN_LEGACY"):
        assert k not in blob, k


def _dummy(n=64):
    buf = (C.c_uint8 * (n + 64))()
    a = C.addressof(buf)
    return buf, C.c_void_p((a + 63) & ~63)


def test_validation_errors_are_synchronous(L):
    from paper_2301_12017_b200._lib import Epilogue, Q4_EALIGN, Q4_EINVAL, Q4_ESHAPE
    keep, p = _dummy()
    # quantize: cols not a multiple of 8
    assert L.q4_quantize_rows(p, 4, 12, 12, 0.0, p, p, None) == Q4_ESHAPE
    assert b"multiples of 8" in L.q4_last_error()
    # quantize: clip not representable in fp16
    assert L.q4_quantize_rows(p, 4, 16, 16, 0.1, p, p, None) == Q4_EINVAL
    # quantize: misaligned x
    assert L.q4_quantize_rows(C.c_void_p(p.value + 2), 4, 16, 16, 0.0, p, p, None) == Q4_EALIGN
    e = Epilogue(kind=1)
    assert L.q4_w4a4_linear(p, p, p, p, 4, 48, 64, C.byref(e), None, 0, None) == Q4_ESHAPE
    assert b"N=48" in L.q4_last_error()
    assert L.q4_w4a4_linear(p, p, p, p, 4, 64, 48, C.byref(e), None, 0, None) == Q4_ESHAPE
    assert L.q4_w4a4_linear(p, p, p, p, 4, 64, 16384, C.byref(e), None, 0, None) == Q4_ESHAPE
    e = Epilogue(kind=9)
    assert L.q4_w4a4_linear(p, p, p, p, 4, 64, 64, C.byref(e), None, 0, None) == Q4_EINVAL
    e = Epilogue(kind=3)  # RESLN without residual
    assert L.q4_w4a4_linear(p, p, p, p, 4, 64, 64, C.byref(e), None, 0, None) == Q4_EINVAL
    assert b"residual" in L.q4_last_error()
    assert L.q4_attention_f16_q4(p, 2, 129, 12, 64, p, p, p, None) == Q4_ESHAPE
    assert L.q4_attention_f16_q4(p, 2, 128, 12, 64, None, p, p, None) == Q4_EINVAL  # ctx_f16 required
    # M = 0 is a no-op that succeeds without touching the device
    e = Epilogue(kind=1)
    assert L.q4_w4a4_linear(p, p, p, p, 0, 64, 64, C.byref(e), None, 0, None) == 0


def test_strategy_names_follow_the_paper():
    """fp16_parts bit i = part q(i+1) runs in FP16 (q4_layer_cfg); names list the quantized
    parts as in PAPER.md:503-504 ("q3" = only the MLP intermediate quantized)."""
    from paper_2301_12017_b200.tune import strategy_name
    assert strategy_name(0) == "qall"
    assert strategy_name(0xF) == "fp16"
    assert strategy_name(0xB) == "q3"
    assert strategy_name(0x5) == "q2q4"
    assert len({strategy_name(m) for m in range(16)}) == 16


def test_layer_structs_match_the_header():
    """The ctypes mirrors of q4_layer_cfg / q4_layer_weights / q4_epilogue carry every field
    the header declares, in order."""
    import re
    from paper_2301_12017_b200 import _lib
    src = open(os.path.join(ROOT, "include", "q4.h")).read()
    body = re.search(r"typedef struct \{([^{}]*?)\} q4_layer_weights;", src, re.S).group(1)
    names = re.findall(r"\*(\w+)", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert tuple(names) == _lib.WEIGHT_FIELDS
    body = re.search(r"typedef struct \{([^{}]*?)\} q4_taps;", src, re.S).group(1)
    assert tuple(re.findall(r"\*(\w+)", re.sub(r"/\*.*?\*/", "", body, flags=re.S))) == _lib.TAP_FIELDS

    def scalar_fields(struct):  # "type a, b;" / "type* a;" declarations, comments removed, in order
        body = re.search(r"typedef struct \{([^{}]*?)\} " + struct + ";", src, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        names = []
        for decl in body.split(";"):
            decl = decl.strip()
            if decl:
                names += [re.sub(r"[*\s]", "", v).split()[-1] if " " in v.strip() else re.sub(r"[*]", "", v).strip()
                          for v in re.sub(r"^(const\s+)?\w+\s*\**", "", decl, count=1).split(",")]
        return [n.strip("* ") for n in names]
    assert scalar_fields("q4_layer_cfg") == [n for n, _ in _lib.LayerCfg._fields_]
    assert scalar_fields("q4_epilogue") == [n for n, _ in _lib.Epilogue._fields_]


def test_workspace_sizes(L):
    """Host-side sizing (no GPU): the row epilogues need exchange slots + counters that grow
    with M and N / tile_n; F16 / I32 need none; the layer / stack workspaces cover them."""
    from paper_2301_12017_b200 import _lib
    ws = L.q4_w4a4_linear_workspace
    assert ws(32768, 3072, 1024, _lib.EPI_F16) == 0 and ws(32768, 3072, 1024, _lib.EPI_I32) == 0
    g = ws(32768, 4096, 1024, _lib.EPI_GELU_Q4)
    r = ws(32768, 1024, 4096, _lib.EPI_RESLN_Q4)
    # [mblocks][ntn][128] x (8 B stats + 4 B max + 8 B asym min/max) + counters: 256 m-blocks,
    # 16 resp. 4 n-blocks
    assert g >= 256 * 16 * 128 * 20 and r >= 256 * 4 * 128 * 20
    assert ws(1024, 4096, 1024, _lib.EPI_GELU_Q4) < g
    # M <= 256: every kind carries the split-K region (tile counters + INT32 partials for
    # N <= 8192 per m-block) at an offset that depends on M only
    f = ws(128, 2304, 768, _lib.EPI_F16)
    assert f >= 8192 * 128 * 4 and f == ws(128, 768, 3072, _lib.EPI_I32)
    assert ws(128, 768, 3072, _lib.EPI_RESLN_Q4) > f and ws(256, 2304, 768, _lib.EPI_F16) > f
    assert ws(257, 2304, 768, _lib.EPI_F16) == 0
    cfg = _lib.LayerCfg(1024, 16, 64, 4096, 1e-12, 0, 0)
    lw = L.q4_encoder_layer_workspace(C.byref(cfg), 256, 128)
    sw = L.q4_encoder_stack_workspace(C.byref(cfg), 256, 128)
    assert lw > g and sw > lw
    assert L.q4_encoder_pipeline_workspace(C.byref(cfg), 256, 128) >= sw + 4 * 256 * 128 * 1024 * 2
