"""Multi-GPU plumbing for the batch axis.

Problems are independent, so ranks shard them with no data-path collective
(weak scaling: every rank solves its own ``per_rank`` problems, global ids
rank * per_rank + b).  The only collectives are for timing and accounting:
the max of the ranks' device times and the sum of their time-DoF.
"""

from __future__ import annotations

import os


def env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def problem_ids(rank: int, world: int, per_rank: int) -> list:
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return [rank * per_rank + b for b in range(per_rank)]


def reduce_time_and_work(elapsed_s: float, dofs: float, device=None):
    """(max elapsed over ranks, sum of time-DoF over ranks); identity when not
    distributed.  Works with nccl (CUDA tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(elapsed_s), float(dofs)
    t = torch.tensor([elapsed_s], dtype=torch.float64, device=device)
    w = torch.tensor([dofs], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t.item()), float(w.item())
