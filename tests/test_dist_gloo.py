"""World-size-2 gloo tests (CPU) of the multi-GPU host logic:
per-rank seeds and profile slices, max-over-ranks timing, sum of units, and the
ordered gather of sharded MDP results.  The MDP part uses the oracle as the
per-rank worker (no GPU here); on GPUs the same slices run libseneca."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth
from paper_2511_13724_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = D.env()
        assert (r, w, lr) == (rank, world, rank)
        # max over ranks / sum over ranks
        times = D.reduce_times([1.0 + rank, 10.0 - rank])
        units = D.reduce_sum([100 * (rank + 1)])
        # sharded MDP sweep: each rank its slice, gathered in rank order
        cols = synth.mdp_profiles(37, seed=4)
        lo, hi = D.profile_slice(37, rank, world)
        rows = O.profiles_from_columns({k: v[lo:hi] for k, v in cols.items()})
        res, _ = O.mdp_sweep(rows, 5)
        full = D.gather_results(res)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), full)
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as f:
            f.write(f"{times[0]} {times[1]} {units[0]} {D.rank_seed(7, rank)}\n")
    finally:
        dist.destroy_process_group()


def test_profile_slices_partition():
    for n in (0, 1, 7, 10_000, 10_001):
        for world in (1, 2, 3, 8):
            sl = [D.profile_slice(n, r, world) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in sl]
            assert max(sizes) - min(sizes) <= 1


def test_rank_seeds_distinct():
    seeds = {D.rank_seed(synth.PERF_SEED, r) for r in range(8)}
    assert len(seeds) == 8 and D.rank_seed(2**64 - 1, 1) == 0


def test_world2_gloo(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import oracle as O
    ref, _ = O.mdp_sweep(O.profiles_from_columns(synth.mdp_profiles(37, seed=4)), 5)
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npy")
        assert got.tobytes() == ref.tobytes()                  # sharded == unsharded, rank order
        t0, t1, u, seed = open(tmp_path / f"r{r}.txt").read().split()
        assert (float(t0), float(t1), float(u)) == (2.0, 10.0, 300.0)
        assert int(seed) == 7 + r


def _shard_worker(rank, world, port, out_dir):
    """attach_shard_peers' exchange with the CUDA calls replaced: each rank
    'shares' a fake handle naming its rank, the mailbox sits at a rank-dependent
    offset in its workspace; every rank must end up with the peers' mailbox
    addresses in shard order and None for itself."""
    import types
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = types.SimpleNamespace(ctx=1000 + rank)
        base = 1 << 40
        attached = {}

        class Fake:
            def __init__(self, h):
                self.h = h

            def data_ptr(self):
                return (1 << 44) * (self.h["rank"] + 1)          # where peer rank's storage maps here

        peers = D.attach_shard_peers(
            g, _share=lambda: (base, {"rank": rank}), _open=Fake,
            _mailbox=lambda ctx: (base + 4096 * (rank + 1), 777),
            _attach=lambda ctx, p: attached.setdefault(ctx, list(p)))
        with open(os.path.join(out_dir, f"s{rank}.txt"), "w") as f:
            f.write(repr((peers, attached[1000 + rank])))
    finally:
        dist.destroy_process_group()


def test_world3_gloo_shard_mailbox_exchange(tmp_path):
    port = _free_port()
    mp.spawn(_shard_worker, args=(3, port, str(tmp_path)), nprocs=3, join=True)
    for r in range(3):
        peers, attached = eval(open(tmp_path / f"s{r}.txt").read())
        assert peers == attached
        want = [None if p == r else (1 << 44) * (p + 1) + 4096 * (p + 1) for p in range(3)]
        assert peers == want


def test_shard_ranges_partition_by_superblock():
    for n in (1, 4096, 4097, 1_281_167, 14_197_122):
        for G in (1, 2, 3, 8):
            rg = D.shard_ranges(n, G)
            assert rg[0][0] == 0 and rg[-1][1] == n and len(rg) == G
            assert all(rg[i][1] == rg[i + 1][0] for i in range(G - 1))
            assert all(lo % 4096 == 0 or lo == n for lo, _ in rg)
