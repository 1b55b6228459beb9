"""Minimal driver for ncu captures: build the pool of a config and run cwb_train twice.
usage: python tools/prof_train.py [R1] [path] [B] [cwb|bernoulli]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cwb_synth as S
from paper_2110_03513_b200 import cwb

name = sys.argv[1] if len(sys.argv) > 1 else "R1"
path = int(sys.argv[2]) if len(sys.argv) > 2 else 0
c = S.CONFIGS[name]
B = int(sys.argv[3]) if len(sys.argv) > 3 else c.B
ds = S.make(c, reps=range(B))
X = torch.as_tensor(ds.X, device="cuda")
Y = torch.as_tensor(ds.Y, device="cuda")
pool = cwb.Pool(X, cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                              degree=c.degree, df=c.df))
pool.set_path(path)
algo = sys.argv[4] if len(sys.argv) > 4 else "cwb"
if algo == "bernoulli":
    Y = torch.as_tensor(S.binary_targets(ds), device="cuda")
for _ in range(2):
    out = pool.train_bernoulli(Y, nu=c.nu, M=c.M) if algo == "bernoulli" else pool.train(Y, nu=c.nu, M=c.M)
pool.status()
torch.cuda.synchronize()
print("ok", name, path, B, float(out["risk_trace"][-1].mean()))
