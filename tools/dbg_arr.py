import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, synth
import paper_2511_13724_b200 as P
st = synth.Stream(14000)
for it in range(40):
    c = synth.random_tiny_ods(st)
    J = len(c["batch"])
    arr = [0 if k == 0 else int(st.u64(1)[0] % 40) for k in range(J)]
    for evict_all in (False, True):
        o = O.ODS(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"], transcript=True, evict_all=evict_all, arrival=arr)
        g = P.ODSContext(c["n_total"], c["batch"], c["target"], c["cap_e"], c["cap_d"], c["cap_a"], c["seed"], evict_tiers=int(evict_all), arrival=arr)
        tr = g.new_transcript()
        rg = g.replay_epochs(max(c["target"]), tr); ro = o.replay_epochs(max(c["target"]))
        torch.cuda.synchronize()
        to = o.transcript(); tg = tr.cpu().numpy().view(np.uint64)
        if not np.array_equal(to, tg) or rg != ro:
            print("MISMATCH it", it, "evict_all", evict_all, c, "arr", arr, "rounds", rg, ro)
            d = np.argwhere(to != tg)
            for (j, e, q) in d[:5]:
                print(" job", j, "epoch", e, "pos", q, "oracle", hex(int(to[j,e,q])), "gpu", hex(int(tg[j,e,q])))
            sys.exit(0)
print("all ok")
