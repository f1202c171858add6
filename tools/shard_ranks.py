"""ONE replay sharded by sample-ID range over W PROCESSES (shard_mode 1, one
shard per process as one process per GPU runs it; here all on cuda:0): each
rank's mailbox is mapped into the others with CUDA IPC by
paper_2511_13724_b200.dist.attach_shard_peers (torch storage sharing, handles
all-gathered over a gloo group), the W round launches exchange pool sizes and
resolved ids device-to-device, and every rank's transcript must equal the
oracle's.  Run by tests/test_gpu_ods.py under a timeout.

    python tools/shard_ranks.py [W] [workload] [scale]
"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, name, scale, seed):
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2511_13724_b200 as P
    import synth
    from paper_2511_13724_b200 import dist as D
    from paper_2511_13724_b200 import seneca as S
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        c = synth.ods_config(name, scale=scale, seed=seed)
        caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
        g = P.ODSContext(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], seed, shards=world,
                         shard_rank=rank, shard_mode=1)
        torch.cuda.synchronize()
        peers = D.attach_shard_peers(g)
        assert peers[rank] is None and all(p for k, p in enumerate(peers) if k != rank)
        tr = g.new_transcript()
        torch.cuda.synchronize()
        dist.barrier()
        rounds = g.replay_epochs(max(c["target"]), tr)
        torch.cuda.synchronize()
        g.sync()
        o = O.ODS(c["n_total"], c["batch"], c["target"], *O.config_capacities(c), seed, transcript=True)
        assert o.replay_epochs(max(c["target"])) == rounds
        assert np.array_equal(tr.cpu().numpy().view(np.uint64), o.transcript()), rank
        assert g.stats()[0].tobytes() == o.stats()[0].tobytes(), rank
        dist.barrier()                      # keep every mailbox mapped until all ranks are done
        print(f"rank {rank}/{world} ok: {c['name']} {rounds} rounds", flush=True)
        g.close()
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    a = sys.argv[1:]
    W = int(a[0]) if a else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(W, port, a[1] if len(a) > 1 else "toy", int(a[2]) if len(a) > 2 else 1, 31),
             nprocs=W, join=True)
    print("all ranks ok", flush=True)
