"""Small invocations of every hand-written kernel family for compute-sanitizer (racecheck / synccheck /
memcheck), one tool per gpurun call (B200_PROFILING.md):

    compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py

fused persistent kernel in CWB (RB = 1 and RB = 2), ACC (ACWB), HC (HCWB) and BERN modes on R0 / R1; the
streaming findBest (k_h1_stream + k_fit_narrow) on R2; the general per-iteration path; the cross-Gram path.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

which = sys.argv[1:] or ["fused", "acc", "hc", "bern", "stream", "general", "gram"]
dev = "cuda:0"


def pool(name, reps):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    p = cwb.Pool(torch.as_tensor(ds.X, device=dev), cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed,
                                                                n_knots=c.n_knots, degree=c.degree, df=c.df))
    return ds, c, p, torch.as_tensor(ds.Y, device=dev)


for w in which:
    if w == "fused":
        for name, reps in (("R0", range(8)), ("R1", range(16)), ("R1", range(300))):  # RB = 1, RB = 2
            ds, c, p, Y = pool(name, reps)
            p.set_path(1)
            p.train(Y, nu=c.nu, M=8)
            p.status()
            p.close()
    elif w == "acc":
        ds, c, p, Y = pool("R1", range(16))
        p.set_path(1)
        p.train_acwb(Y, nu=c.nu, M=8)
        p.status()
        p.close()
    elif w == "hc":
        for B in (16, 200):  # one 512-thread CTA per replication / two 256-thread CTAs per SM
            ds, c, p, Y = pool("R1", range(B))
            p.set_path(1)
            vm = torch.as_tensor(S.validation_mask(c.n), device=dev)
            p.train_hcwb(Y, vm, nu=0.1, gamma=0.5, pat0=2, M=12)
            p.status()
            p.close()
    elif w == "bern":
        ds, c, p, Y = pool("R1", range(16))
        p.set_path(1)
        p.train_bernoulli(torch.as_tensor(S.binary_targets(ds), device=dev), nu=c.nu, M=8)
        p.status()
        p.close()
    elif w == "stream":
        for B in (1, 3):
            ds, c, p, Y = pool("R2", range(B))
            p.set_narrow(0)
            p.find_best(Y - Y.mean(1, keepdim=True))
            p.status()
            p.close()
    elif w == "general":
        ds, c, p, Y = pool("R1", range(40))
        p.set_path(2)
        p.train(Y, nu=c.nu, M=3)
        p.status()
        p.close()
    elif w == "gram":
        ds, c, p, Y = pool("R1", range(40))
        p.set_path(3)
        p.train(Y, nu=c.nu, M=6)
        p.status()
        p.close()
    torch.cuda.synchronize()
    print("ok", w, flush=True)
