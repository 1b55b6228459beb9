"""Phase timing of the cross-Gram path (cwb_set_path 3) against the direct per-iteration path, CUDA events:
    python tools/gram_timing.py R3 R4
fresh pool M = 0 (cross-Gram build + s^[0]), cached pool M = 0 (s^[0] only), cached pool M (all iterations)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402


def ev_time(fn, reps=3):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


for name in sys.argv[1:] or ["R3"]:
    ds = S.make(name)
    c = ds.cfg
    X = torch.as_tensor(ds.X, device="cuda")
    Y = torch.as_tensor(ds.Y, device="cuda")
    cfg = cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots, degree=c.degree,
                     df=c.df)
    res = {"workload": name}

    def fresh_m0():
        p = cwb.Pool(X, cfg)
        p.set_path(3)
        p.train(Y, nu=c.nu, M=0)
        p.status()
        p.close()
    res["init_ms"] = ev_time(lambda: cwb.Pool(X, cfg).close())
    res["fresh_M0_ms"] = ev_time(fresh_m0)
    p = cwb.Pool(X, cfg)
    p.set_path(3)
    p.train(Y, nu=c.nu, M=0)
    res["cached_M0_ms"] = ev_time(lambda: p.train(Y, nu=c.nu, M=0))
    res["cached_M_ms"] = ev_time(lambda: p.train(Y, nu=c.nu, M=c.M))
    p.status()
    p.close()

    def full_step():
        q = cwb.Pool(X, cfg)
        q.set_path(3)
        q.train(Y, nu=c.nu, M=c.M)
        q.close()
    res["step_ms"] = ev_time(full_step)
    res["xgram_build_ms"] = res["fresh_M0_ms"] - res["cached_M0_ms"] - res["init_ms"]
    res["iterations_ms"] = res["cached_M_ms"] - res["cached_M0_ms"]
    res["evals_per_s"] = c.K * c.n * c.B * c.M / (res["step_ms"] * 1e-3)
    print(json.dumps(res), flush=True)
