"""One cwb_train call of M iterations on a rung's full launch (for ncu launch lists of the per-iteration path).
    python tools/prof_iter.py R3 3"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R3"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ds = S.make(name)
c = ds.cfg
pool = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed,
                                                                  n_knots=c.n_knots, degree=c.degree, df=c.df,
                                                                  batch_hint=c.B))
Y = torch.as_tensor(ds.Y, device="cuda")
for _ in range(2):
    out = pool.train(Y, nu=c.nu, M=M)
pool.status()
torch.cuda.synchronize()
print("ok", name, M, pool.launches())
