"""Write oracle results for the full-size ODS configs to tests/golden/.

This script calls only oracle/ (and synth/ for the workload description): the
stored values are the oracle's, never the CUDA path's.  GPU tests and bench.py
compare the device replay against these files (per job-epoch counters and
digests, eviction/refill totals, a hash of the final residency/seen/consumer
state).

    python tests/golden/make_oracle_golden.py imagenet1k [seed [scale [evict_all]]]
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def caps_for(c):
    return O.config_capacities(c)


def state_hash(tier, seen, cons):
    h = hashlib.sha256()
    h.update(tier.tobytes()); h.update(seen.tobytes()); h.update(cons.tobytes())
    return h.hexdigest()


def main(name, seed, scale=1, evict_all=False):
    c = synth.ods_config(name, scale=scale, seed=seed)
    ce, cd, ca = caps_for(c)
    t0 = time.time()
    o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, seed, evict_all=evict_all)
    rounds = o.replay_epochs(max(c["target"]))
    dt = time.time() - t0
    st, ev, rf = o.stats()
    tier, seen, cons = o.state()
    out = dict(
        config=c["name"], seed=seed, n_total=c["n_total"], batch=c["batch"], target=c["target"],
        caps=[ce, cd, ca], evict_tiers=int(evict_all), rounds=int(rounds), evicted=int(ev), refilled=int(rf),
        stats=[[dict(served=[int(v) for v in st[j, e]["served"]], subst=[int(v) for v in st[j, e]["subst"]],
                     req_hits=[int(v) for v in st[j, e]["req_hits"]], digest=str(int(st[j, e]["digest"])))
                for e in range(st.shape[1])] for j in range(st.shape[0])],
        state_sha256=state_hash(tier, seen, cons),
        oracle_seconds=round(dt, 1),
        generator="tests/golden/make_oracle_golden.py (oracle/ only)",
    )
    path = os.path.join(HERE, f"oracle_{c['name'].replace('/', '_s')}_seed{seed}{'_evictall' if evict_all else ''}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, f"{dt:.1f}s", rounds, "rounds")


if __name__ == "__main__":
    name = sys.argv[1]
    seed = int(sys.argv[2], 0) if len(sys.argv) > 2 else synth.PERF_SEED
    scale = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    evict_all = len(sys.argv) > 4 and sys.argv[4] in ("1", "all", "evict_all")
    main(name, seed, scale, evict_all)
