"""Edge-configuration probe: every training entry point on tiny / degenerate shapes, GPU against the oracle.
usage: python tools/probe_edges.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from oracle import oracle as O
from paper_2110_03513_b200 import cwb
import cwb_synth as S

def dev(a, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")

cases = [  # (n, K, B, ns, degree, knots, df)
    (2, 1, 1, 2, 1, 0, 2.0), (3, 1, 2, 3, 1, 0, 2.0), (5, 2, 3, 5, 1, 1, 2.5), (40, 1, 1, 6, 2, 2, 3.0),
    (300, 1, 1, 17, 3, 4, 4.0), (1000, 2, 1, 30, 3, 20, 5.0), (64, 3, 33, 8, 3, 3, 4.0)]
for (n, K, B, ns, dg, nk, df) in cases:
    rng = np.random.default_rng(n + K + B)
    X = rng.uniform(-1, 2, (K, n))
    Y = np.sin(2 * X[0])[None, :] + 0.3 * rng.standard_normal((B, n))
    ocfg = O.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df)
    gcfg = cwb.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df)
    tag = f"n={n} K={K} B={B} ns={ns} deg={dg} knots={nk} df={df}"
    try:
        po = O.Pool(X, ocfg, O.MODE_BINNED)
    except O.OracleError as e:
        try:
            pg = cwb.Pool(dev(X), gcfg); pg.status(); print(tag, "ORACLE", e.name, "GPU ok (mismatch)")
        except cwb.CwbError as g:
            print(tag, "both reject", e.name, g.name)
        continue
    res = []
    for path in (0, 1, 2):
        try:
            pg = cwb.Pool(dev(X), gcfg)
            pg.set_path(path)
            out = pg.train(dev(Y), nu=0.2, M=12)
            pg.status()
            g = {k: v.cpu().numpy() for k, v in out.items()}
            o = po.train(Y, nu=0.2, M=12)
            ok = (g["k_trace"] == o.k_trace).all() and np.allclose(g["risk_trace"], o.risk_trace, rtol=1e-9, atol=1e-14)
            res.append(f"train{path}:{'ok' if ok else 'MISMATCH'}")
            for name, fn in (("acwb", lambda: pg.train_acwb(dev(Y), nu=0.2, gamma=0.01, M=12)),
                             ("hcwb", lambda: pg.train_hcwb(dev(Y), dev(S.validation_mask(n), torch.uint8), nu=0.2, gamma=0.05, pat0=2, M=12)),
                             ("bern", lambda: pg.train_bernoulli(dev((Y > np.median(Y)).astype(float)), nu=0.2, M=12))):
                try:
                    fn(); pg.status(); res.append(f"{name}{path}:ok")
                except cwb.CwbError as e:
                    res.append(f"{name}{path}:{e.name}")
            k, th, sse = pg.find_best(dev(Y[:1] - Y[:1].mean()))
            pg.status()
            ko = po.find_best((Y[:1] - Y[:1].mean())[0])[0]
            res.append(f"fb{path}:{'ok' if int(k[0]) == ko else 'MISMATCH'}")
            pg.close()
        except cwb.CwbError as e:
            res.append(f"path{path}:{e.name}:{str(e)[:60]}")
    print(tag, " ".join(res))
