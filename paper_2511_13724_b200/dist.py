"""Multi-GPU plumbing: one process per GPU, torch.distributed for
rendezvous, the mailbox mapping of a sharded replay and the timing reduction.

The north_star partitions the path two ways:
  * independent problems -- every rank replays its own instance of the
    workload (seed + rank) and sweeps its own MDP profiles (weak scaling, no
    data-path collective);
  * ONE replay partitioned by sample-ID range: rank r is shard
    r (shard_mode 1).  The per-round exchange (every shard's pool sizes, the
    ids each shard resolved) runs inside the round kernels, device to device:
    each rank's mailbox is mapped into every other rank with CUDA IPC (torch's
    storage sharing) and the kernels store into the peers' mailboxes over
    NVLink (attach_shard_peers).  torch.distributed only carries the handles.
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


def attach_shard_peers(g, group=None, _share=None, _open=None, _mailbox=None, _attach=None):
    """Shard mode 1 (one shard per rank): map every rank's shard mailbox into this
    process and attach them to the context of `g` (a paper_2511_13724_b200.ODSContext
    whose workspace tensor is g.ws).  The mailbox lives inside the workspace; its
    CUDA IPC handle is the workspace storage's (torch storage sharing), plus the
    mailbox's byte offset in it.  Returns the peers' device pointers (own: None)."""
    import torch.distributed as dist
    import torch
    from . import seneca
    # (the _hooks replace the CUDA calls in the CPU test of this exchange)
    share = _share or (lambda: (g.ws.untyped_storage().data_ptr(), g.ws.untyped_storage()._share_cuda_()))
    open_ = _open or (lambda h: torch.UntypedStorage._new_shared_cuda(*h))
    ptr, nbytes = (_mailbox or seneca.shard_mailbox)(g.ctx)
    base, handle = share()
    mine = (dist.get_rank(group), handle, ptr - base, nbytes)
    infos = [None] * dist.get_world_size(group)
    dist.all_gather_object(infos, mine, group=group)
    peers, keep = [], []
    for rk, h, o, _ in sorted(infos, key=lambda t: t[0]):
        if rk == dist.get_rank(group):
            peers.append(None)
            continue
        st = open_(h)
        keep.append(st)
        peers.append(st.data_ptr() + o)
    (_attach or seneca.shard_attach)(g.ctx, peers)
    g._peer_storages = keep
    return peers


def shard_ranges(n_total: int, shards: int):
    """The sample-ID range [lo, hi) of each shard (superblocks of 4096 ids split
    into ceil(NS / G)-superblock runs; seneca.h shards) -- host mirror used by
    tests and reports."""
    ns = -(-n_total // 4096)
    per = -(-ns // shards)
    out = []
    for g in range(shards):
        lo, hi = min(ns, g * per), min(ns, (g + 1) * per)
        out.append((min(n_total, lo * 4096), min(n_total, hi * 4096)))
    return out
