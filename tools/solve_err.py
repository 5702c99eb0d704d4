import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2003_07504_b200 as ils
g = np.load("tests/golden/golden.npz")
worst_abs = worst_rel = 0.0
for key in g.files:
    if key.startswith("solve_") and key.endswith("_u"):
        k = key[:-2]
        lam, c = g[k + "_lamc"]
        f, mx, my = g[k + "_f"], g[k + "_mx"], g[k + "_my"]
        plan = ils.make_plan(f.shape[0], f.shape[1], lam, c, f)
        u = ils.solve_ls(plan, f, mx, my, precision="fp32")
        e = np.max(np.abs(u - g[key]))
        worst_abs = max(worst_abs, e)
        worst_rel = max(worst_rel, e / max(1.0, np.max(np.abs(g[key]))))
print("fp32 solve_ls vs goldens: max abs", worst_abs, "max rel", worst_rel)
