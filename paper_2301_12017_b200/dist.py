"""Batch-sharded data parallelism for the W4A4 encoder.

Sequences are independent, so the path shards by batch with no collective in the data
path: rank r of W takes its contiguous slice of the global batch, holds full weight
replicas, and runs the same CUDA graph.  The only cross-rank operations are host-side
plumbing: a barrier around the timed region and a max-reduction of the per-rank device
time (the job finishes when the slowest rank does).  torch.distributed supplies the
process group (NCCL on GPUs, gloo in the CPU tests)."""
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
