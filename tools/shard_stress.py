"""Stress: many emulated sharded replays (G = 2, 4, 8) against the oracle (counters)."""
import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle as O, synth
import paper_2511_13724_b200 as P
from paper_2511_13724_b200 import seneca as S
res = {}
for name, scale in (("toy", 1), ("imagenet1k", 64)):
    seed = 12
    c = synth.ods_config(name, scale=scale, seed=seed)
    ce, cd, ca = O.config_capacities(c)
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed)
    ro = o.replay_epochs(max(c["target"]))
    st_o = o.stats()[0].tobytes()
    for G in (2, 4, 8):
        bad = 0; errs = set()
        for it in range(10):
            g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, shards=G)
            r = g.replay_epochs(max(c["target"]))
            torch.cuda.synchronize()
            try:
                g.sync()
                ok = all(g.stats(k)[0].tobytes() == st_o for k in range(G))
            except Exception as e:
                ok = False; errs.add(str(e)[:80])
            bad += not ok
            g.close()
        print(name, G, "bad", bad, "/10", errs, flush=True)
