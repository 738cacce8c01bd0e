"""Batch-sharded data parallelism for the W4A4 encoder.

Sequences are independent, so the path shards by batch with no collective in the data
path: rank r of W takes its contiguous slice of the global batch, holds full weight
replicas, and runs the same CUDA graph.  The one data collective is the gather of the
outputs after the last layer (`OutputGather`); the rest is host-side plumbing: a barrier
around the timed region and a max-reduction of the per-rank device time (the job
finishes when the slowest rank does).  torch.distributed supplies the process group
(NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests)."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_ranks():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(global_batch: int, rank: int, world: int):
    """Contiguous slice [start, start + count) of the global batch owned by `rank`.
    Every sequence is owned by exactly one rank; sizes differ by at most one."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity if none)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


class OutputGather:
    """The one collective of the batch-sharded path (north_star: "no collective in the hot
    path beyond an NCCL gather of outputs"): every rank's final hidden states
    [B_r * S, h] are gathered, in rank order, into the global [B * S, h] -- mode "full" --
    or only the [CLS] row (token 0) of each sequence, [B, h] -- mode "cls", the input of a
    BERT classification head.  Rank r's rows land at [r * B_r, (r+1) * B_r): the gathered
    tensor is the single-GPU output of the same global batch (shards are equal-sized here).

    Buffers are allocated once (graph- and replay-friendly); `__call__` is stream-ordered
    and does not synchronize.  Without a process group: the local tensor itself (no
    collective); with one, the collective runs at any world size (size 1 included, so a
    single-GPU box exercises the NCCL path)."""

    def __init__(self, B: int, S: int, h: int, mode: str = "cls", device=None, dtype=torch.float16):
        if mode not in ("cls", "full"):
            raise ValueError(f"gather mode {mode!r} (expected 'cls' or 'full')")
        self.B, self.S, self.h, self.mode = B, S, h, mode
        self.pg = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size() if self.pg else 1
        rows = B if mode == "cls" else B * S
        self.local = torch.empty(rows, h, dtype=dtype, device=device) if mode == "cls" else None
        self.out = torch.empty(self.world * rows, h, dtype=dtype, device=device) if self.pg else None

    @property
    def bytes_per_rank(self) -> int:
        rows = self.B if self.mode == "cls" else self.B * self.S
        return rows * self.h * 2

    def __call__(self, hidden: torch.Tensor) -> torch.Tensor:
        if tuple(hidden.shape) != (self.B * self.S, self.h):
            raise ValueError(f"gather: hidden {tuple(hidden.shape)} != ({self.B * self.S}, {self.h})")
        if self.mode == "cls":
            self.local.copy_(hidden.view(self.B, self.S, self.h)[:, 0])
            src = self.local
        else:
            src = hidden
        if not self.pg:
            return src
        dist.all_gather_into_tensor(self.out, src.contiguous())
        return self.out
