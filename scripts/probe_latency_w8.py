"""BERT-base W8A8 layer stack at batch 1 x seq 128 (latency config), eager (profiling helper:
A/B timing against scripts/probe_latency.py, the W4A4 stack)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
L = int(sys.argv[1]) if len(sys.argv) > 1 else 12
base = dict(synth.BERT["base"])
enc = q4.W8A8Encoder(base, [synth.layer_params(base, l, "bert") for l in range(L)], device="cuda")
x = torch.from_numpy(synth.hidden(128, 768, "input", 0)).cuda()
o = torch.empty_like(x)
for _ in range(5):
    enc.forward(x, o, 1, 128)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    enc.forward(x, o, 1, 128)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"L": L, "w8a8_eager_ms": e0.elapsed_time(e1) / 20}))
