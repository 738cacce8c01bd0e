"""The batch-sharded launcher's collective on the GPU: an NCCL process
group on the B200 (world size 1 -- gpurun and the round-end tiers have one GPU; the
multi-rank ordering is covered by the gloo tests in test_dist_cpu.py).  The encoder's
output goes through OutputGather's NCCL all-gather in both modes and must come back
unchanged; the [CLS] mode must pick token 0 of every sequence."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2301_12017_b200 import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    yield dev
    dist.destroy_process_group()


def test_nccl_output_gather_encoder(nccl_group):
    import paper_2301_12017_b200 as q4
    from paper_2301_12017_b200 import dist as qd
    dev = nccl_group
    assert dist.get_backend() == "nccl"
    cfg = dict(synth.BERT["base"])
    B, S, L = 4, 128, 2
    enc = q4.W4A4Encoder(cfg, [synth.layer_params(cfg, l, "bert") for l in range(L)], device=dev)
    start, count = qd.shard(B, 0, 1)
    assert (start, count) == (0, B)
    x = torch.from_numpy(np.concatenate([synth.hidden(S, cfg["hidden"], "input", b) for b in range(B)])).to(dev)
    out = torch.empty_like(x)
    enc.forward(x, out, B, S)
    for mode in ("cls", "full"):
        g = qd.OutputGather(B, S, cfg["hidden"], mode=mode, device=dev)
        assert g.pg and g.world == 1
        got = g(out)
        torch.cuda.synchronize()
        want = out.view(B, S, -1)[:, 0] if mode == "cls" else out
        assert got.data_ptr() != out.data_ptr()  # the collective's own buffer
        assert torch.equal(got, want)
    qd.barrier()
    assert qd.max_over_ranks(3.5, dev) == 3.5
