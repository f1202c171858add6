"""One MDP sweep (n profiles, 1 % grid, grid written) for ncu captures.
    python tools/profile_mdp.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2511_13724_b200 as P  # noqa: E402
import synth  # noqa: E402
from paper_2511_13724_b200 import seneca as S  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
rows = S.profiles_from_columns(synth.mdp_profiles(n))
for _ in range(2):
    P.mdp_sweep_device(rows, 1, want_grid=True)
torch.cuda.synchronize()
