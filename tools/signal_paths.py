"""Coupled replays (A churn, evict-all, cold start) with the round launch and
signal path chosen by the environment (SENECA_ROUND_CLUSTER / SENECA_DSMEM_SIGNALS,
read once per process), cut into launches of random length, vs the oracle:
transcripts, counters and bitmaps.  Run by tests/test_gpu_ods.py in a subprocess.

    SENECA_ROUND_CLUSTER=0 python tools/signal_paths.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2511_13724_b200 as P  # noqa: E402
import synth  # noqa: E402


def main():
    st = synth.Stream(4242)
    n_cfg = 0
    for name, scale, kw in (("toy", 1, {}), ("imagenet1k", 64, {}), ("imagenet1k", 64, {"evict_all": True}),
                            ("imagenet1k", 64, {"cold": True})):
        c = synth.ods_config(name, scale=scale, seed=77)
        ce, cd, ca = O.config_capacities(c)
        o = O.ODS(c["n_total"], c["batch"], c["target"], ce, cd, ca, 77, transcript=True, **kw)
        g = P.ODSContext(c["n_total"], c["batch"], c["target"], ce, cd, ca, 77,
                         evict_tiers=int(kw.get("evict_all", False)), cold_start=int(kw.get("cold", False)))
        tr = g.new_transcript()
        total = 0
        while g.view().active_mask:
            k = int(st.u64(1)[0] % np.uint64(300)) + 1
            done = g.replay_rounds(k, tr)
            total += done
            if done < k:
                break
        torch.cuda.synchronize()
        g.sync()
        assert total == o.replay_epochs(max(c["target"])), (name, kw)
        assert np.array_equal(tr.cpu().numpy().view(np.uint64), o.transcript()), (name, kw)
        st_o, ev_o, rf_o = o.stats()
        st_g, ev_g, rf_g = g.stats()
        assert (ev_g, rf_g) == (ev_o, rf_o) and st_g.tobytes() == st_o.tobytes(), (name, kw)
        for a, b in zip(g.state(), o.state()):
            np.testing.assert_array_equal(a, b)
        g.close()
        n_cfg += 1
    print(f"signal paths ok: {n_cfg} coupled replays, SENECA_ROUND_CLUSTER={os.environ.get('SENECA_ROUND_CLUSTER', '-')}"
          f" SENECA_DSMEM_SIGNALS={os.environ.get('SENECA_DSMEM_SIGNALS', '-')}", flush=True)


if __name__ == "__main__":
    main()
