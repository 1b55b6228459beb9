"""GPU parity of the cross-Gram path (cwb_set_path 3) against the oracle's Alg. 1
supp.: the same iterates as the direct path up to rounding (s_k updated through Z_k^T Z_k*, r^T r by its
exact expansion), so the selected-learner sequences must be identical except at verified near ties (tie
rule 1e-12) and the traces / parameters agree within 1e-9 over all iterations -- which also bounds the drift
of the incremental updates."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import cfg_of, close, follow_parity, gpu_cfg_of  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def gram_train(name, reps=None, M=None):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.set_path(3)
    out = pg.train(dev(ds.Y), nu=c.nu, M=M or c.M)
    pg.status()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    return ds, pg, g


@pytest.mark.parametrize("name", ["R0", "R1"])
def test_gram_all_replications_tie_following(name):
    ds, pg, g = gram_train(name)
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(g, po, ds.Y, c.nu, c.M, f"{name} gram")
    assert fol.sum() <= max(1, 0.01 * c.M * c.B)
    # aggregation: predict(X) with the path-3 parameters reproduces the oracle's fit (the residuals are never
    # formed on this path, so this checks theta_agg against the model itself)
    pred = pg.predict(dev(ds.X), dev(g["offset"]), dev(g["theta_agg"])).cpu().numpy()
    o = po.train(ds.Y, nu=c.nu, M=c.M, threads=8)
    same = (o.k_trace == g["k_trace"]).all(0)
    ok, e = close(pred[same], o.f[same], 1e-9, scale=np.abs(o.f).max())
    assert ok, e
    pg.close()


def test_gram_r2_sampled_replications():
    ds, pg, g = gram_train("R2", reps=[0, 1, 2, 3, 500, 1023])
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(g, po, ds.Y, c.nu, c.M, "R2 gram", threads=6)
    assert fol.sum() <= 2
    pg.close()


@pytest.mark.slow
def test_gram_r3_full_launch():
    # the R3 bench launch (B = 512), replications 0-7 and the last, all 200 iterations
    ds, pg, g = gram_train("R3")
    c = ds.cfg
    reps = [0, 1, 2, 3, 4, 5, 6, 7, 511]
    sub = {k: (v[:, reps] if v.ndim == 2 and k != "theta_agg" else v[reps]) for k, v in g.items()}
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(sub, po, ds.Y[reps], c.nu, c.M, "R3 gram B=512", threads=len(reps))
    assert fol.sum() <= 2
    pg.close()


@pytest.mark.slow
def test_gram_r4_full_launch():
    # the R4 launch (B = 64, n = 1,000,000, K = 84, n* = 1000), replications 0-3, all 200 iterations
    ds, pg, g = gram_train("R4")
    c = ds.cfg
    reps = [0, 1, 2, 3]
    sub = {k: (v[:, reps] if v.ndim == 2 and k != "theta_agg" else v[reps]) for k, v in g.items()}
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(sub, po, ds.Y[reps], c.nu, c.M, "R4 gram B=64", threads=len(reps))
    assert fol.sum() <= 2
    pg.close()


def test_gram_equals_direct_path_and_deterministic():
    ds = S.make("R1", reps=range(64))
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    res = {}
    for p in (2, 3, 3):
        pg.set_path(p)
        out = pg.train(dev(ds.Y), nu=c.nu, M=c.M)
        pg.status()
        res.setdefault(p, []).append({k: v.cpu().numpy() for k, v in out.items()})
    a, b, b2 = res[2][0], res[3][0], res[3][1]
    for k in b:
        assert (b[k] == b2[k]).all(), k   # run to run bitwise
    assert (a["k_trace"] == b["k_trace"]).mean() > 0.99
    same = (a["k_trace"] == b["k_trace"]).all(0)
    ok, e = close(b["theta_agg"][same], a["theta_agg"][same], 1e-10, scale=np.abs(a["theta_agg"]).max())
    assert ok, e
    ok, e = close(b["risk_trace"][:, same], a["risk_trace"][:, same], 1e-11)
    assert ok, e
    pg.close()


def test_gram_edge_cases_and_errors():
    rng = np.random.default_rng(5)
    X = rng.uniform(0, 1, (3, 80))
    Y = rng.standard_normal((5, 80))
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=4))
    pg.set_path(3)
    out = pg.train(dev(Y), nu=0.0, M=4)       # nu = 0: nothing moves
    pg.status()
    assert (out["theta_agg"].cpu().numpy() == 0).all()
    r = out["risk_trace"].cpu().numpy()
    assert np.allclose(r, r[0], rtol=0, atol=0)
    out = pg.train(dev(Y), nu=0.1, M=0)       # M = 0: offset only
    assert np.allclose(out["offset"].cpu().numpy(), Y.mean(1), rtol=1e-13)
    with pytest.raises(cwb.CwbError) as e:    # the other training variants do not take path 3
        pg.train_acwb(dev(Y), M=3)
    assert e.value.name == "CWB_EUNSUPPORTED"
    Yb = Y.copy()
    Yb[2, 5] = np.inf
    pg.train(dev(Yb), nu=0.1, M=2)
    with pytest.raises(cwb.CwbError) as e:
        pg.status()
    assert e.value.name == "CWB_ENONFINITE"


@pytest.mark.parametrize("seed,n,K,degree,n_knots,ns_fixed", [
    (11, 1237, 5, 3, 20, 0),     # odd n (the pairs' index rows start at every 2-byte alignment), sqrt rule
    (12, 4001, 7, 2, 6, 300),    # u16 bins, degree 2, few knots (wide windows), several bin tiles per pair
    (13, 997, 4, 1, 9, 40),      # degree 1
    (14, 70001, 3, 3, 20, 0),    # 32-bit row ids, n* = 265
])
def test_gram_joint_build_edge_shapes(seed, n, K, degree, n_knots, ns_fixed):
    """The cross-Gram blocks come from the joint bin counts of learner pairs (k_gram_joint): ragged n,
    clamped learners (a feature with few distinct values: n*_k < n*), both index widths and row-id widths,
    B-spline degrees 1-3 -- path 3 against the oracle's Alg. 1, tie rule 1e-12."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((K, n))
    X[1] = rng.integers(0, 7, n).astype(np.float64)          # 7 distinct values: clamped n*_k
    X[K - 1] = np.round(X[0] * 3.0) / 3.0 + 0.01 * X[K - 1]   # strongly dependent on learner 0: dense count cells
    B, M, nu = 6, 40, 0.1
    Y = np.sin(X[0]) + 0.5 * X[2] ** 2 + 0.3 * rng.standard_normal((B, n))
    kw = dict(n_star_rule=2 if ns_fixed else 0, n_star_fixed=ns_fixed, n_knots=n_knots, degree=degree, df=4.0)
    pg = cwb.Pool(dev(X), cwb.Config(**kw))
    pg.set_path(3)
    out = pg.train(dev(Y), nu=nu, M=M)
    pg.status()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    po = O.Pool(X, O.Config(**kw), O.MODE_BINNED)
    fol = follow_parity(g, po, Y, nu, M, f"gram joint n={n} K={K} deg={degree}")
    assert fol.sum() <= 1
    pg.close()


@pytest.mark.slow
def test_gram_equals_direct_path_r3_all_replications():
    # every replication of the R3 bench launch (B = 512, 200 iterations): the cross-Gram path and the direct
    # per-iteration path (itself oracle-checked on replications 0-7, 255, 511) select the same learners except
    # where the two runs' SSE gap is a tie within 1e-12; traces and parameters agree to rounding
    ds = S.make("R3")
    c = ds.cfg
    gc = gpu_cfg_of(c)
    gc.batch_hint = c.B
    pg = cwb.Pool(dev(ds.X), gc)
    res = {}
    for p in (2, 3):
        pg.set_path(p)
        out = pg.train(dev(ds.Y), nu=c.nu, M=c.M)
        pg.status()
        res[p] = {k: v.cpu().numpy() for k, v in out.items()}
    a, b = res[2], res[3]
    same = (a["k_trace"] == b["k_trace"]).all(0)
    print(f"[parity] R3 gram vs direct: {int(same.sum())} of {c.B} replications identical over {c.M} iterations")
    for r in np.nonzero(~same)[0]:   # a divergence must start at a near tie of the direct run's SSEs
        m = int(np.nonzero(a["k_trace"][:, r] != b["k_trace"][:, r])[0][0])
        assert abs(a["sse_trace"][m, r] - b["sse_trace"][m, r]) <= 1e-12 * abs(a["sse_trace"][m, r]) * 10, (r, m)
    assert same.mean() >= 0.99
    ok, e = close(b["theta_agg"][same], a["theta_agg"][same], 1e-9, scale=np.abs(a["theta_agg"]).max())
    assert ok, e
    ok, e = close(b["risk_trace"][:, same], a["risk_trace"][:, same], 1e-10)
    assert ok, e
    pg.close()
