"""GPU parity over the learner configuration space the C ABI accepts (include/cwb.h cwb_config):
B-spline degree 1..3, inner-knot counts 0..28 (d = n_knots + degree + 1 <= 32), few bins
(n* = 2, 3, 5: rank-deficient Z^T Z, reading G19) and df targets near the feasible edge.
Where the oracle rejects a configuration (df outside (nullity, d]) the GPU must reject
it with the same status; otherwise the fused and per-iteration training paths and the
streaming findBest agree with the oracle (agreement rules of tests/parity_util.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, TIE_RTOL, close  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"
CASES = [  # (degree, n_knots, n*, df)
    (1, 0, 3, 2.0), (1, 5, 40, 3.0), (2, 0, 9, 2.5), (2, 12, 60, 5.0), (3, 0, 12, 3.5),
    (3, 28, 100, 8.0), (1, 20, 37, 5.0), (2, 20, 37, 5.0), (3, 4, 5, 4.0), (3, 20, 2, 5.0),
    (3, 20, 3, 5.0), (2, 3, 5, 5.0),
]


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(out):
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def data(seed, n=900, K=4, B=6):
    rng = np.random.default_rng(seed)
    X = np.stack([rng.uniform(-2, 3, n) if k % 2 == 0 else rng.standard_normal(n) for k in range(K)])
    Y = np.stack([np.cos(X[0] * (1 + 0.2 * b)) + 0.5 * X[1] ** 2 * (b % 2) + 0.3 * rng.standard_normal(n)
                  for b in range(B)])
    return X, Y


@pytest.mark.parametrize("degree,n_knots,ns,df", CASES)
def test_learner_config_matches_oracle(degree, n_knots, ns, df):
    X, Y = data(degree * 100 + n_knots + ns)
    ocfg = O.Config(n_star_rule=2, n_star_fixed=ns, degree=degree, n_knots=n_knots, df=df)
    gcfg = cwb.Config(n_star_rule=2, n_star_fixed=ns, degree=degree, n_knots=n_knots, df=df)
    try:
        po = O.Pool(X, ocfg, O.MODE_BINNED)
    except O.OracleError as e:
        with pytest.raises(cwb.CwbError) as g:
            pg = cwb.Pool(dev(X), gcfg)
            pg.status()
        assert g.value.name == "CWB_" + e.name
        return
    pg = cwb.Pool(dev(X), gcfg)
    pg.status()
    if n_knots + degree + 1 > 2:  # d <= 2: no penalty, every lambda meets the target (oracle: 1)
        lam_g = pg.lam()
        assert close(lam_g, po.lam, 1e-8)[0], (lam_g, po.lam)
    for path in (1, 2):
        pg.set_path(path)
        g = host(pg.train(dev(Y), nu=0.1, M=40))
        pg.status()
        o, fol = po.train_follow(Y, g["k_trace"], tie_rtol=TIE_RTOL, nu=0.1, M=40, threads=6)
        print(f"[parity] ties followed: {int(fol.sum())} over {fol.size} replications (tie rule {TIE_RTOL:g})")
        assert (o.k_trace == g["k_trace"]).all(), f"path {path}"
        for key, ref in (("theta_agg", o.theta_agg), ("sse_trace", o.sse_trace), ("risk_trace", o.risk_trace)):
            ok, e = close(g[key], ref, RTOL, scale=np.abs(ref).max())
            assert ok, f"path {path} {key} {e}"
        if path == 2:  # prediction on new points, in and outside the training range
            Xn = np.concatenate([X[:, :200] * 0.9 + 0.05, X[:, :40] * 2.5], axis=1)
            pred = pg.predict(dev(Xn), dev(g["offset"]), dev(g["theta_agg"])).cpu().numpy()
            opred = po.predict(Xn, g["offset"], g["theta_agg"])
            ok, e = close(pred, opred, RTOL, scale=np.abs(opred).max())
            assert ok, f"predict {e}"
    # streaming findBest, one column
    R = Y[:1] - Y[:1].mean(1, keepdims=True)
    pg.set_narrow(0)
    k, th, sse = (t.cpu().numpy() for t in pg.find_best(dev(R)))
    ko, tho, sseo, _, gap = po.find_best(R[0])
    if k[0] != ko:
        assert gap / sseo <= TIE_RTOL
    else:
        assert close(sse[0], sseo, RTOL)[0]
        assert close(th[0], tho, RTOL, scale=np.abs(tho).max())[0]
    pg.close()


def test_bin_count_limit():
    # the largest pool n* (12288) trains and matches the oracle's findBest; one more bin is rejected
    rng = np.random.default_rng(31)
    n = 40000
    X = np.stack([rng.uniform(-1, 1, n), rng.standard_normal(n)])
    Y = np.sin(3 * X[:1]) + 0.2 * rng.standard_normal((1, n))
    pg = cwb.Pool(dev(X), cwb.Config(n_star_rule=2, n_star_fixed=12288, n_knots=20))
    po = O.Pool(X, O.Config(n_star_rule=2, n_star_fixed=12288, n_knots=20), O.MODE_BINNED)
    assert (pg.n_star_k() == po.nsk).all()
    R = Y - Y.mean(1, keepdims=True)
    k, th, sse = (t.cpu().numpy() for t in pg.find_best(dev(R)))
    ko, tho, sseo, _, gap = po.find_best(R[0])
    assert k[0] == ko and close(sse[0], sseo, RTOL)[0]
    pg.close()
    with pytest.raises(cwb.CwbError) as e:
        cwb.Pool(dev(X), cwb.Config(n_star_rule=2, n_star_fixed=12289, n_knots=20))
    assert e.value.name == "CWB_EUNSUPPORTED"
