"""A few cwb_find_best calls on one residual column (for ncu launch lists): python tools/fb_once.py R3"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

c = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "R3"]
ds = S.make(c, reps=[0])
pool = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed,
                                                                  n_knots=c.n_knots))
R = torch.as_tensor(ds.Y - ds.Y.mean(1, keepdims=True), device="cuda")
for _ in range(4):
    pool.find_best(R)
pool.status()
torch.cuda.synchronize()
print("ok", c.name)
