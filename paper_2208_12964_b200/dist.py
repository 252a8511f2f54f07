"""Multi-GPU plumbing for the slice stack (one process per GPU).

SURVEY.md §8(e): the 2D-stack configuration shards by slice with no
communication during iterations; cone-beam MART (C3/C4) does not shard (the
reference's update within a view is sequential), so it runs replicas only.
torch.distributed is used for rendezvous, the barrier around the timed region,
the max-over-ranks timing reduction and the optional end gather of fields —
never inside a sweep.
"""
from __future__ import annotations

import os
from typing import Tuple

import numpy as np


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of n items for `rank` (strong scaling of a
    fixed stack: slices [lo, hi) on this GPU)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


def rank_seed(base: int, rank: int) -> int:
    """Seed of rank `rank`'s own stack under weak scaling (distinct phantoms)."""
    return base + 1000 * rank


def max_over_ranks(values, device=None):
    """Element-wise max over ranks of a list of floats (the timing rule:
    a multi-GPU number is the slowest rank's device time)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.cpu()]


def gather_stack(local: np.ndarray, n_total: int, rank: int, world: int, device=None):
    """End-of-run gather of slice-sharded fields to rank 0: local holds this
    rank's shard(n_total) rows; returns the (n_total, ...) stack on rank 0 and
    None elsewhere. One collective after the iterations, none during."""
    import torch
    import torch.distributed as dist
    lo, hi = shard(n_total, rank, world)
    assert local.shape[0] == hi - lo
    row = int(np.prod(local.shape[1:]))
    cap = (n_total + world - 1) // world
    buf = torch.zeros((cap, row), dtype=torch.float32, device=device)
    buf[: hi - lo] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float32).reshape(hi - lo, row)).to(buf)
    if world == 1:
        return buf[:n_total].cpu().numpy().reshape((n_total,) + local.shape[1:])
    parts = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, parts, dst=0)
    if rank != 0:
        return None
    rows = [parts[r][: shard(n_total, r, world)[1] - shard(n_total, r, world)[0]] for r in range(world)]
    return torch.cat(rows).cpu().numpy().reshape((n_total,) + local.shape[1:])
