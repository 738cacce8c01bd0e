"""O-10 free-running drift.  The L-layer stack is
"parity unpinned": once a layer's fp16 output differs from the oracle's by an ulp, a
requant code can flip and the two sides see different inputs from then on, so the stack
cannot be compared element by element.  What CAN be compared is how far the two
free-running stacks drift: per layer, the fraction of INT4 codes that differ, the
largest code difference and the relative L2 error of the fp16 hidden state, with the
GPU and the oracle each feeding its own outputs forward (the CUDA-
graph encoder; synthetic BERT weights).

Bounds (R22): every layer is parity-green teacher-forced (test_gpu_parity), so
the free-running gap can only come from rounding-order differences that flip codes
sitting within an fp16 ulp of a rounding boundary; such a flip moves the code by one.
How far those flips spread is a property of the model, not of the kernels: with random-init
weights the layer map is expanding, and any ulp-level difference grows layer by layer until
the two trajectories are decorrelated (measured: ~0.2% code flips after layer 0, tens of
percent by layer 5).  So the deeper layers are compared against a CONTROL that involves no
GPU arithmetic after layer 0: the oracle restarted from the GPU's layer-0 output.  The
control and the GPU stack start from the same perturbation; if the kernels added error of
their own in later layers, the GPU's drift would run ahead of the control's.  The test
asserts that no code differs by more than 1 in layer 0, that layer 0 flips < 1% of the codes,
and that at every layer the GPU's flip rate and hidden-state error stay within a small
factor of the control's.
With Q4_DRIFT_REPORT=<path> it also writes the per-layer report as JSON."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as orc
from paper_2301_12017_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q4():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2301_12017_b200 as q4
    q4.lib()
    return q4


def _oracle_weights(p):
    w = {}
    for k in ("wqkv", "wo", "w1", "w2"):
        w[k], w["s" + k[1:]] = orc.quantize_rows(p[k])
    for k in ("bqkv", "bo", "b1", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"):
        w[k] = p[k]
    return w


def drift_report(q4, size, L, B, S, seed="drift"):
    cfg = dict(synth.BERT[size])
    h = cfg["hidden"]
    layers = [synth.layer_params(cfg, l, seed) for l in range(L)]
    x = synth.hidden(B * S, h, seed + "_x")
    # GPU: explicit per-layer calls (== q4_encoder_stack bit for bit, test_gpu_parity)
    gw = [q4.quantize_layer(p) for p in layers]
    xd = torch.from_numpy(x).cuda()
    ghq, ghs = q4.quantize_rows(xd)
    gh = xd
    # oracle: its own weights (O-3) and its own outputs fed forward
    ow = [_oracle_weights(p) for p in layers]
    ohq, ohs = orc.quantize_rows(x)
    oh = x
    ch = chq = chs = None  # control: the oracle fed the GPU's layer-0 output
    rep = []
    for l in range(L):
        o = q4.encoder_layer(cfg, gw[l], B, S, gh, ghq, ghs)
        gh, ghq, ghs = o["h_out"], o["hq_out"], o["hs_out"]
        r = orc.encoder_layer(cfg, ow[l], B, S, oh, ohq, ohs)
        oh, ohq, ohs = r["h_out"], r["hq_out"], r["hs_out"]
        torch.cuda.synchronize()
        g16, gq = gh.cpu().numpy().astype(np.float64), orc.unpack_int4(ghq.cpu().numpy(), h)
        o16, oq = oh.astype(np.float64), orc.unpack_int4(ohq, h)
        if l == 0:
            ch, chq, chs = gh.cpu().numpy(), ghq.cpu().numpy(), ghs.cpu().numpy()
        else:
            c = orc.encoder_layer(cfg, ow[l], B, S, ch, chq, chs)
            ch, chq, chs = c["h_out"], c["hq_out"], c["hs_out"]
        c16, cq = ch.astype(np.float64), orc.unpack_int4(chq, h)
        d = np.abs(gq.astype(np.int32) - oq.astype(np.int32))
        dc = np.abs(cq.astype(np.int32) - oq.astype(np.int32))
        rep.append({"layer": l,
                    "code_flip_rate": float((d != 0).mean()),
                    "max_code_diff": int(d.max()),
                    "rel_l2_h": float(np.linalg.norm(g16 - o16) / np.linalg.norm(o16)),
                    "max_abs_h": float(np.abs(g16 - o16).max()),
                    "scale_rel_max": float(np.abs(ghs.cpu().numpy() / ohs - 1).max()),
                    "control_code_flip_rate": float((dc != 0).mean()),
                    "control_rel_l2_h": float(np.linalg.norm(c16 - o16) / np.linalg.norm(o16))})
    return rep


@pytest.mark.parametrize("size,L,B", [("base", 12, 2), ("large", 24, 1)])
def test_free_running_stack_drift(q4, size, L, B):
    rep = drift_report(q4, size, L, B, 128)
    path = os.environ.get("Q4_DRIFT_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"model": size, "layers": L, "batch": B, "seq": 128, "per_layer": rep}) + "\n")
    assert rep[0]["max_code_diff"] <= 1, rep[0]
    assert rep[0]["code_flip_rate"] < 1e-2, rep[0]
    for r in rep[1:]:
        # the GPU stack adds fresh ulp-level differences at every layer, the control only at
        # layer 0: allow a small factor plus an absolute floor for the early layers
        assert r["code_flip_rate"] <= 3.0 * r["control_code_flip_rate"] + 0.01, r
        assert r["rel_l2_h"] <= 3.0 * r["control_rel_l2_h"] + 0.01, r
