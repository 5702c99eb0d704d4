import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2003_07504_b200 as ils
from paper_2003_07504_b200 import _runtime as rt
params = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0, iters=int(os.environ.get("ITERS", "4")))
rng = np.random.default_rng(3)
x = torch.from_numpy(rng.random((3, 1080, 1920))).to("cuda", torch.float32)
a = ils.smooth_batch(x, params)
c = ils.smooth_batch(x[1:2].clone(), params)
d = (c[0] - a[1]).abs()
print("maxdiff", d.max().item(), "count", (d > 0).sum().item())
idx = torch.nonzero(d > 0)
print(idx[:10].tolist())
for B in (1, 3):
    print(B, rt.get_plan(B, 1080, 1920, params.c_params(), 0, 0).info)
