"""Event time of cwb_init (I1-I8 pool build) on a config, and algorithmic HBM bytes of the
elementwise init kernels.  usage: python tools/init_timing.py [R4] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cwb_synth as S
from paper_2110_03513_b200 import cwb

name = sys.argv[1] if len(sys.argv) > 1 else "R4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = S.CONFIGS[name]
ds = S.make(c, reps=[0])
X = torch.as_tensor(ds.X, device="cuda")
cfg = cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots, degree=c.degree, df=c.df)
cwb.Pool(X, cfg).close()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    p = cwb.Pool(X, cfg)
    e1.record()
    p.status()
    ts.append(e0.elapsed_time(e1))
    p.close()
K, n = ds.X.shape
print(f"{name} K={K} n={n} cwb_init {min(ts):.3f} ms (min of {reps}); X = {K * n * 8 / 1e6:.0f} MB")
