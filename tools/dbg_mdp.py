import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_mdp as T
rows = T.table4_rows()
print("N", rows["n_total"][:5], len(rows))
for g in [int(a) for a in sys.argv[1:]]:
    try:
        res, grid = T.run_gpu(rows, g)
        print(g, "ok", res["p_e"][:4])
    except Exception as e:
        print(g, "ERR", str(e)[:200]); break
