"""Runs one small invocation of every kernel family and saves every output (for the schedule-perturbation
test, tests/test_gpu_jitter.py):   CWB_LIB=<lib> python tools/det_run.py out.npz"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

dev = "cuda:0"
res = {}


def pool(name, reps):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    p = cwb.Pool(torch.as_tensor(ds.X, device=dev), cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed,
                                                                n_knots=c.n_knots, degree=c.degree, df=c.df))
    return ds, c, p, torch.as_tensor(ds.Y, device=dev)


def keep(tag, out):
    for k, v in out.items():
        res[f"{tag}/{k}"] = v.cpu().numpy()


for tag, name, B in (("fused_rb1", "R1", 100), ("fused_rb2", "R1", 300), ("fused_r0", "R0", 8)):
    ds, c, p, Y = pool(name, range(B))
    p.set_path(1)
    keep(tag, p.train(Y, nu=c.nu, M=60))
    p.status(); p.close()
ds, c, p, Y = pool("R1", range(40))
p.set_path(1)
keep("acc", p.train_acwb(Y, nu=c.nu, M=60))
p.status()
keep("bern", p.train_bernoulli(torch.as_tensor(S.binary_targets(ds), device=dev), nu=c.nu, M=60))
p.status()
p.set_path(2)
keep("general", p.train(Y, nu=c.nu, M=20))
p.set_path(3)
keep("gram", p.train(Y, nu=c.nu, M=60))
p.status(); p.close()
for B in (40, 200):
    ds, c, p, Y = pool("R1", range(B))
    p.set_path(1)
    vm = torch.as_tensor(S.validation_mask(c.n), device=dev)
    keep(f"hc{B}", p.train_hcwb(Y, vm, nu=0.1, gamma=0.5, pat0=2, M=80))
    p.status(); p.close()
for name, B in (("R2", 1), ("R2", 3), ("R3", 1)):
    ds, c, p, Y = pool(name, range(B))
    p.set_narrow(0)
    k, th, sse = p.find_best(Y - Y.mean(1, keepdim=True))
    keep(f"stream_{name}_{B}", {"k": k, "theta": th, "sse": sse})
    p.status(); p.close()
torch.cuda.synchronize()
np.savez(sys.argv[1], **res)
print("saved", len(res), "arrays to", sys.argv[1], "with", cwb.LIB_PATH)
