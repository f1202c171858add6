"""One sample-ID-range-sharded replay with ONE SHARD PER CONTEXT (shard_mode 1),
the way one process per GPU runs it, here with G contexts on one device:
each context's mailbox is attached to the others (seneca_shard_attach) and the
G round launches run concurrently on G streams, exchanging through each
other's mailboxes.  Every shard's transcript must equal the oracle's.
Run by tests/test_gpu_ods.py in a subprocess under a timeout.

    python tools/shard_contexts.py [G] [workload] [scale]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2511_13724_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2511_13724_b200 import seneca as S  # noqa: E402


def main(G=2, name="toy", scale=1, seed=21):
    c = synth.ods_config(name, scale=scale, seed=seed)
    caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
    streams = [torch.cuda.Stream() for _ in range(G)]
    ctxs = [P.ODSContext(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], seed, shards=G,
                         shard_rank=g, shard_mode=1, stream=streams[g]) for g in range(G)]
    torch.cuda.synchronize()
    boxes = [S.shard_mailbox(x.ctx)[0] for x in ctxs]
    for x in ctxs:
        S.shard_attach(x.ctx, boxes)
    trs = [x.new_transcript() for x in ctxs]
    torch.cuda.synchronize()
    rounds = [x.replay_epochs(max(c["target"]), tr) for x, tr in zip(ctxs, trs)]   # G concurrent launches
    torch.cuda.synchronize()
    for x in ctxs:
        x.sync()
    o = O.ODS(c["n_total"], c["batch"], c["target"], *O.config_capacities(c), seed, transcript=True)
    ro = o.replay_epochs(max(c["target"]))
    assert all(r == ro for r in rounds), (rounds, ro)
    t_o = o.transcript()
    st_o = o.stats()[0].tobytes()
    for g, (x, tr) in enumerate(zip(ctxs, trs)):
        assert np.array_equal(tr.cpu().numpy().view(np.uint64), t_o), g
        assert x.stats()[0].tobytes() == st_o, g
    print(f"sharded one-context-per-shard replay ok: G={G} {c['name']} {ro} rounds", flush=True)


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 2, a[1] if len(a) > 1 else "toy", int(a[2]) if len(a) > 2 else 1)
