import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_12017_b200 as q4
from paper_2301_12017_b200 import synth
B, S, H = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 128, 16)
qkv = torch.from_numpy(synth.hidden(B * S, 3 * H * 64, "pa_qkv")).cuda()
for _ in range(3): q4.attention_f16_q4(qkv, B, S, H)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(10): q4.attention_f16_q4(qkv, B, S, H)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"attn_us": e0.elapsed_time(e1) / 10 * 1e3}))
