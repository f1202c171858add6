"""Find the first random tiny cold-start config where the GPU replay and the oracle differ."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, synth
import paper_2511_13724_b200 as P
st = synth.Stream(16000)
for it in range(50):
    c = synth.random_tiny_ods(st)
    for evict_all, baseline in ((False, False), (True, False), (False, True)):
        o = O.ODS(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"], transcript=True, evict_all=evict_all, baseline=baseline, cold=True)
        g = P.ODSContext(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"], evict_tiers=int(evict_all), sampler=int(baseline), cold_start=1)
        tr = g.new_transcript()
        rg = g.replay_epochs(max(c["target"]), tr); ro = o.replay_epochs(max(c["target"]))
        torch.cuda.synchronize()
        to = o.transcript(); tg = tr.cpu().numpy().view(np.uint64)
        if not np.array_equal(to, tg) or rg != ro:
            print("MISMATCH it", it, "evict_all", evict_all, "baseline", baseline, c, "rounds", rg, ro)
            for (j, e, q) in np.argwhere(to != tg)[:6]:
                print(" job", j, "epoch", e, "pos", q, "oracle", hex(int(to[j,e,q])), "gpu", hex(int(tg[j,e,q])))
            print(" tiers oracle", list(o.state()[0]))
            print(" tiers gpu   ", list(g.state()[0]))
            sys.exit(0)
print("all ok")
