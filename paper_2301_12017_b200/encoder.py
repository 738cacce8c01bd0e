"""a8: the L-layer W4A4 BERT encoder: one q4_encoder_stack call per
forward -- initial activation quantize + L x [QKV, attention, attn-out, FFN1, FFN2] --
optionally captured once into a CUDA graph and replayed ("we enable CUDA graph in our
inference pipeline to minimize such overhead").  Marshalling only."""
from __future__ import annotations

import ctypes as C

import torch

from . import ops
from ._lib import LayerWeights, check, lib


class W4A4Encoder:
    bits = 4

    def __init__(self, cfg: dict, layers: list, device="cuda", fp16_parts: int = 0, asym: bool = False):
        """cfg: BERT dims (hidden, heads, head_dim, ffn, ln_eps); layers: per-layer fp16
        parameter dicts (synth.layer_params) -- quantized on the device here (offline).
        fp16_parts: the per-part quantization strategy (q4_layer_cfg; 0 = qall).
        asym: asymmetric activation quantization throughout (NEXT-3, q4_layer_cfg.asym_acts)."""
        self.cfg = dict(cfg)
        self.cfg["fp16_parts"] = fp16_parts
        self.cfg["asym_acts"] = int(asym)
        self.device = torch.device(device)
        self.weights = [ops.quantize_layer(p, self.device, bits=self.bits, fp16_parts=fp16_parts, asym=asym)
                        for p in layers]
        i8 = self.bits == 8
        self._ws_fn = lib().q4_encoder_stack_w8a8_workspace if i8 else lib().q4_encoder_stack_workspace
        self._stack_fn = lib().q4_encoder_stack_w8a8 if i8 else lib().q4_encoder_stack
        self.L = len(self.weights)
        self._lw = (LayerWeights * self.L)(*[ops.layer_weights(w) for w in self.weights])
        self._lc = ops.layer_cfg(self.cfg)
        self._ws = {}  # (B, S) -> workspace; kept alive: a captured graph holds raw pointers into it
        self.graph = None
        self._graph_key = None

    def sibling(self):
        """A second encoder over the same device weights, with its own workspaces and graph
        (e.g. the same model captured at another batch size)."""
        other = object.__new__(type(self))
        other.__dict__.update(self.__dict__)
        other._ws, other.graph, other._graph_key = {}, None, None
        other._pws = {}
        return other

    def workspace(self, B: int, S: int) -> torch.Tensor:
        ws = self._ws.get((B, S))
        if ws is None:
            n = self._ws_fn(C.byref(self._lc), B, S)
            ws = self._ws[(B, S)] = torch.zeros(max(n, 1), dtype=torch.uint8, device=self.device)
        return ws

    def forward(self, h_in: torch.Tensor, h_out: torch.Tensor, B: int, S: int):
        """h_in / h_out: fp16 [B*S, hidden], CUDA tensors or (pinned) CPU tensors -- with
        host tensors the H2D / D2H copies happen inside the C call (end-to-end path)."""
        ws = self.workspace(B, S)
        check(self._stack_fn(C.byref(self._lc), self._lw, self.L, B, S,
                                     C.c_void_p(h_in.data_ptr()), C.c_void_p(h_out.data_ptr()),
                                     C.c_void_p(ws.data_ptr()), ws.numel(),
                                     C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return h_out

    def serve(self, h_in: list, h_out: list, B: int, S: int):
        """Pipelined end-to-end serving (q4_encoder_pipeline, W4A4 only): lists of host fp16
        [B*S, hidden] tensors (pinned for overlap); batch i's upload and batch i-1's download
        overlap batch i's forward.  Stream-ordered on the current stream."""
        if self.bits != 4:
            raise ValueError("serve(): the pipelined entry runs the W4A4 stack")
        if len(h_in) != len(h_out):
            raise ValueError("serve(): h_in and h_out lengths differ")
        # one zero-filled workspace per shape (the row-epilogue counters sit at M-dependent offsets)
        pws = getattr(self, "_pws", {})
        self._pws = pws
        if (B, S) not in pws:
            n = lib().q4_encoder_pipeline_workspace(C.byref(self._lc), B, S)
            pws[(B, S)] = torch.zeros(max(n, 1), dtype=torch.uint8, device=self.device)
        ws = pws[(B, S)]
        pin = (C.c_void_p * len(h_in))(*[t.data_ptr() for t in h_in])
        pout = (C.c_void_p * len(h_out))(*[t.data_ptr() for t in h_out])
        check(lib().q4_encoder_pipeline(C.byref(self._lc), self._lw, self.L, B, S, pin, pout, len(h_in),
                                        C.c_void_p(ws.data_ptr()), ws.numel(),
                                        C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return h_out

    def capture(self, h_in: torch.Tensor, h_out: torch.Tensor, B: int, S: int, warmup: int = 1):
        """Capture forward(h_in -> h_out) (device buffers) into a CUDA graph."""
        self.workspace(B, S)
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.forward(h_in, h_out, B, S)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward(h_in, h_out, B, S)
        self.graph = g
        # the graph replays into this shape's workspace and these buffers: keep them alive
        self._graph_key = (B, S, h_in, h_out)
        return g

    def replay(self):
        if self.graph is None:
            raise RuntimeError("replay(): no graph captured (call capture() first)")
        self.graph.replay()


class W8A8Encoder(W4A4Encoder):
    """The W8A8 baseline encoder (the paper's INT8 comparison point,
    PAPER.md:496-502): the same stack with 8-bit codes (q4_encoder_stack_w8a8)."""
    bits = 8
