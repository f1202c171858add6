"""Multi-GPU plumbing: one process per GPU, torch.distributed for
rendezvous and the timing reduction only -- the hot path has no data-path
collective.

The north_star partitions the path into independent problems:
  * ODS: every rank replays its own instance of the workload (seed + rank),
    i.e. replicas across GPUs (weak scaling); a single replay's round chain is
    latency-bound and would only slow down if sample-ID ranges were split
    across GPUs (two all-gathers per round cost more than the
    round itself);
  * MDP: the profile set is split into contiguous slices, one per rank (or, for
    weak scaling, every rank sweeps its own profile set).
"""
from __future__ import annotations

import os

import numpy as np


def env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def rank_seed(seed: int, rank: int) -> int:
    """Seed of rank `rank`'s independent replay instance (seed + rank, 64-bit)."""
    return (seed + rank) & 0xFFFFFFFFFFFFFFFF


def profile_slice(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n profiles for `rank`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def reduce_times(values, group=None, device=None):
    """Max over ranks of per-rank elapsed times (seconds): the job is as slow as
    its slowest rank.  Returns a list of floats."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


def reduce_sum(values, group=None, device=None):
    """Sum over ranks (units processed)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.tolist()


def gather_results(local: np.ndarray, group=None, device=None) -> np.ndarray:
    """Concatenate equal-dtype per-rank result rows in rank order (variable
    lengths allowed); used to assemble a sharded MDP sweep's results."""
    import torch
    import torch.distributed as dist
    raw = np.ascontiguousarray(local).view(np.uint8).reshape(-1)
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return local.copy()
    world = dist.get_world_size()
    n = torch.tensor([raw.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = int(max(int(s) for s in sizes))
    buf = torch.zeros(m, dtype=torch.uint8, device=device)
    buf[:raw.size] = torch.from_numpy(raw).to(device)
    outs = [torch.zeros(m, dtype=torch.uint8, device=device) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    parts = [o[:int(s)].cpu().numpy() for o, s in zip(outs, sizes)]
    return np.concatenate(parts).view(local.dtype)
