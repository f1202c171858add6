"""Time alternative builds of the MDP sweep against each other (same inputs):
    python tools/mdp_variants.py lib_a.so lib_b.so ...
Each library is loaded with ctypes; results and grid must be byte-identical to
the first library's.  Device timing with CUDA events over 20 launches."""
import ctypes as C
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_13724_b200 import seneca as S  # noqa: E402

n = int(os.environ.get("MDP_N", "10000"))
rows = S.profiles_from_columns(synth.mdp_profiles(n))
d_prof = torch.from_numpy(np.ascontiguousarray(rows).view(np.uint8)).cuda()
ns = S.mdp_num_splits(1)
ref = None
for path in sys.argv[1:]:
    L = C.CDLL(os.path.abspath(path))
    f = L.seneca_mdp_sweep
    f.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
    f.restype = C.c_int
    d_res = torch.zeros(n * 48, dtype=torch.uint8, device="cuda")
    for want_grid in (True, False):
        d_grid = torch.empty((n, ns), dtype=torch.float64, device="cuda") if want_grid else None
        gp = d_grid.data_ptr() if want_grid else None
        for _ in range(3):
            assert f(d_prof.data_ptr(), n, 1, d_res.data_ptr(), gp, None) == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            f(d_prof.data_ptr(), n, 1, d_res.data_ptr(), gp, None)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        h = hashlib.sha256(d_res.cpu().numpy().tobytes())
        if want_grid:
            h.update(d_grid.cpu().numpy().tobytes())
        dig = h.hexdigest()[:16]
        if ref is None and want_grid:
            ref = dig
        tag = "grid" if want_grid else "argmax"
        ok = (dig == ref) if want_grid else ""
        print(f"{os.path.basename(path):28s} {tag:6s} {us:8.1f} us  {n * ns / us / 1e3:7.1f} G split/s  "
              f"{n * ns * 8 / us / 1e3 if want_grid else 0:7.0f} GB/s  {dig} {ok}", flush=True)
