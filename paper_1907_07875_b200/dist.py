"""Multi-GPU plumbing for the batch-sharded GFT (one process per GPU, torch.distributed).

The fast GFT of independent signals shards along the batch with no data-path collective
(SURVEY §8(e)); every rank builds the same plan (the planner is deterministic) and
transforms its own rows.  Only timing needs a collective: the MAX over ranks.
"""
from __future__ import annotations

import os


def dist_env():
    """(world_size, rank, local_rank) from the torchrun environment (defaults: 1, 0, 0)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_rows(batch: int, rank: int, world: int):
    """Contiguous row range [start, start+count) of `rank` (sizes differ by at most 1)."""
    if world < 1 or not (0 <= rank < world) or batch < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(batch, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (e.g. ms per step) over all ranks; identity when not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(device=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        if device is not None and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()
