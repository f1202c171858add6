"""Drive a bounded ODS replay (and optionally the MDP sweep) for ncu captures.

    python tools/profile_ods.py imagenet1k 2000 [--mdp] [--plain]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_13724_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2511_13724_b200 import seneca as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "imagenet1k"
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
c = synth.ods_config(name, seed=synth.PERF_SEED)
caps = S.split_capacities(c["n_total"], c["s_data"], c["m_num"], c["m_den"], c["cache_bytes"], *c["split"])
g = P.ODSContext(c["n_total"], c["batch"], c["target"], caps[0], caps[1], caps[2], c["seed"])
g.profile(0 if "--plain" in sys.argv else 3)   # event timing + in-kernel phase counters (--plain: none)
g.replay_rounds(rounds)
torch.cuda.synchronize()
ph = g.phase_cycles()
print("rounds", rounds, "phase cycles", ph.tolist())
print({k: v for k, v in g.profile_read().items() if v["launches"]})
if "--mdp" in sys.argv:
    rows = S.profiles_from_columns(synth.mdp_profiles(10_000))
    P.mdp_sweep_device(rows, 1, want_grid=True)
    torch.cuda.synchronize()
