import ctypes as C, os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import test_gpu_mdp as T
rows = T.to_dev_rows(T.table4_rows())
n = len(rows)
d_prof = torch.from_numpy(np.ascontiguousarray(rows).view(np.uint8)).cuda()
L = C.CDLL(os.path.abspath(sys.argv[1])); f = L.seneca_mdp_sweep
f.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
for cnt in (1, 2, 4, 5, 8, 54):
    d_res = torch.zeros(48 * cnt, dtype=torch.uint8, device="cuda")
    d_grid = torch.empty((cnt, 5151), dtype=torch.float64, device="cuda")
    rc = f(d_prof.data_ptr(), cnt, 1, d_res.data_ptr(), d_grid.data_ptr(), None)
    try:
        torch.cuda.synchronize(); print(sys.argv[1], cnt, "ok", rc)
    except Exception as e:
        print(sys.argv[1], cnt, "FAILS", str(e)[:80]); sys.exit(0)
