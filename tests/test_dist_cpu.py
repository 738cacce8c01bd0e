"""Multi-process host logic of the batch-sharded path (gloo, world_size 2, CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_12017_b200 import dist as qd
from paper_2301_12017_b200 import synth


def test_shard_partitions_the_batch():
    for gb in (1, 7, 256, 1000):
        for w in (1, 2, 3, 4, 8):
            got = [qd.shard(gb, r, w) for r in range(w)]
            assert sum(c for _, c in got) == gb
            assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(w - 1))
            assert max(c for _, c in got) - min(c for _, c in got) <= 1
    with pytest.raises(ValueError):
        qd.shard(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = qd.env_ranks()
        start, count = qd.shard(6, r, w)
        # each rank generates only its own sequences; seeds are per sequence
        x = np.concatenate([synth.hidden(16, 64, "input", b) for b in range(start, start + count)])
        qd.barrier()
        m = qd.max_over_ranks(10.0 * (r + 1))
        q.put((r, start, count, x, m))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shards_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.concatenate([synth.hidden(16, 64, "input", b) for b in range(6)])
    got = np.concatenate([x for _, _, _, x, _ in res])
    assert np.array_equal(got, full)  # shards reassemble the single-rank global batch
    assert all(m == 20.0 for *_, m in res)  # max over ranks seen by every rank
    assert [(s, c) for _, s, c, _, _ in res] == [(0, 3), (3, 3)]


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, S, h = 3, 4, 8
        start, count = qd.shard(B * world, rank, world)
        loc = torch.from_numpy(np.concatenate([synth.hidden(S, h, "input", b) for b in range(start, start + count)]))
        got = {m: qd.OutputGather(B, S, h, m)(loc).clone().numpy() for m in ("cls", "full")}
        with pytest.raises(ValueError):
            qd.OutputGather(B, S, h, "full")(loc[:-1])
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_output_gather():
    """The gathered outputs equal the single-rank global batch (full) and its [CLS] rows."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.concatenate([synth.hidden(4, 8, "input", b) for b in range(6)])
    for _, got in res:  # every rank holds the whole gathered output
        assert np.array_equal(got["full"], full)
        assert np.array_equal(got["cls"], full[::4])


def test_output_gather_single_process():
    B, S, h = 2, 3, 4
    x = torch.arange(B * S * h, dtype=torch.float16).view(B * S, h)
    assert torch.equal(qd.OutputGather(B, S, h, "full")(x), x)
    assert torch.equal(qd.OutputGather(B, S, h, "cls")(x), x[::S])
    with pytest.raises(ValueError):
        qd.OutputGather(B, S, h, "rows")


def _strong_worker(rank, world, port, q):
    """bench.py's strong-scaling data path with a stub forward: global batch GB split over the
    ranks (qd.shard), a per-sequence forward (mixes tokens within a sequence, so a shard that
    split a sequence or misordered them would show), the [CLS] / full gather in rank order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        GB, S, h = 8, 4, 8
        start, B = qd.shard(GB, rank, world)
        x = torch.from_numpy(np.concatenate([synth.hidden(S, h, "input", b) for b in range(start, start + B)]))
        y = _stub_forward(x, B, S, h)
        q.put((rank, {m: qd.OutputGather(B, S, h, m)(y).clone().numpy() for m in ("cls", "full")},
                  qd.max_over_ranks(float(B))))
    finally:
        dist.destroy_process_group()


def _stub_forward(x, B, S, h):
    xs = x.float().view(B, S, h)
    return (xs.cumsum(1) * 0.5 + xs.mean(1, keepdim=True)).half().view(B * S, h)


def test_two_rank_gloo_strong_scaling_stub_forward():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    GB, S, h = 8, 4, 8
    x = torch.from_numpy(np.concatenate([synth.hidden(S, h, "input", b) for b in range(GB)]))
    ref = _stub_forward(x, GB, S, h).numpy()
    for _, got, m in res:
        assert np.array_equal(got["full"], ref)  # sharded + gathered == one process, whole batch
        assert np.array_equal(got["cls"], ref[::S])
        assert m == GB // world
