"""GPU parity of the per-learner n* clamp (reading N1):
n*_k = min(n*, #distinct values of feature k) -- from k_distinct's hash set in shared memory
(n* <= 8192) or in a global table (larger n*) -- and everything built on it: the design points
and index vectors (bit-exact), G and lambda, and training / findBest on every path, against
the oracle on tied features."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, TIE_RTOL, close  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(out):
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def tied(seed, n, spec):
    """One feature per entry: an int -> that many distinct values (random levels), 'c' -> continuous,
    'z' -> values in {-1.5, -0.0, +0.0, 2.25} (3 distinct), ('h', m) -> a heavy value on n/3 rows
    and m other values."""
    rng = np.random.default_rng(seed)
    rows = []
    for s in spec:
        if s == "c":
            rows.append(rng.standard_normal(n))
        elif s == "z":
            rows.append(rng.choice([-1.5, -0.0, 0.0, 2.25], n))
        elif isinstance(s, tuple):
            x = rng.choice(rng.uniform(-4, 9, s[1]), n)
            x[: n // 3] = 0.5
            rows.append(x)
        else:
            x = rng.choice(rng.uniform(-4, 9, s), n)
            x[:s] = rng.permutation(np.unique(x[s:]).tolist() + [x[0]] * (s - len(np.unique(x[s:]))))[:s]
            rows.append(x)
    return np.stack(rows)


@pytest.mark.parametrize("seed,n,ns,spec,df", [
    (0, 2000, None, [7, "c", "z", 45, 44], 2.5),          # sqrt rule: n* = 45
    (1, 5000, 300, [("h", 150), 299, 300, 301, "c"], 5.0),
    (2, 30000, 10000, [6000, "c", ("h", 9000)], 5.0),     # n* > 8192: global hash table
])
def test_n_star_k_and_pool_match_oracle(seed, n, ns, spec, df):
    X = tied(seed, n, spec)
    rule, fixed = (0, 0) if ns is None else (2, ns)
    po = O.Pool(X, O.Config(n_star_rule=rule, n_star_fixed=fixed, n_knots=10, df=df), O.MODE_BINNED)
    pg = cwb.Pool(dev(X), cwb.Config(n_star_rule=rule, n_star_fixed=fixed, n_knots=10, df=df))
    pg.status()
    nsk = pg.n_star_k()
    assert (nsk == po.nsk).all(), (nsk, po.nsk)
    assert (nsk == np.minimum(po.n_star, [len(np.unique(x)) for x in X])).all()
    P = host(pg.pool())
    assert (P["idx"].astype(np.int64) == po.idx).all()
    assert (P["z"] == po.z).all()
    ok, e = close(P["G"], po.G, 1e-12, scale=np.abs(po.G).max())
    assert ok, e
    assert close(pg.lam(), po.lam, 1e-8)[0]
    pg.close()


@pytest.mark.parametrize("path", [1, 2])
def test_train_on_tied_features_matches_oracle(path):
    n = 3000  # n* = 55
    X = tied(3, n, [5, "c", 12, ("h", 40), 54])
    rng = np.random.default_rng(3)
    Y = np.stack([np.sin(X[0]) + 0.2 * X[2] + 0.3 * np.cos(X[4]) + 0.5 * rng.standard_normal(n) for _ in range(10)])
    cfg = dict(n_knots=8, df=3.5)  # 5 distinct values: rank-5 G
    po = O.Pool(X, O.Config(**cfg), O.MODE_BINNED)
    pg = cwb.Pool(dev(X), cwb.Config(**cfg))
    pg.set_path(path)
    g = host(pg.train(dev(Y), nu=0.1, M=60))
    pg.status()
    o, fol = po.train_follow(Y, g["k_trace"], tie_rtol=TIE_RTOL, nu=0.1, M=60, threads=8)
    print(f"[parity] ties followed: {int(fol.sum())} over {fol.size} replications (tie rule {TIE_RTOL:g})")
    assert (o.k_trace == g["k_trace"]).all()
    for key, ref in (("theta_agg", o.theta_agg), ("sse_trace", o.sse_trace), ("risk_trace", o.risk_trace)):
        ok, e = close(g[key], ref, RTOL, scale=np.abs(ref).max())
        assert ok, f"{key} {e}"
    # prediction on new points (tied values, values between and outside the training levels)
    Xn = np.concatenate([X[:, :300], X[:, :300] + 0.37, X[:, :50] * 3.0 - 2.0], axis=1)
    pred = pg.predict(dev(Xn), dev(g["offset"]), dev(g["theta_agg"])).cpu().numpy()
    opred = po.predict(Xn, g["offset"], g["theta_agg"])
    ok, e = close(pred, opred, RTOL, scale=np.abs(opred).max())
    assert ok, f"predict {e}"
    # streaming findBest on one column
    R = Y[:1] - Y[:1].mean(1, keepdims=True)
    pg.set_narrow(0)
    k, th, sse = (t.cpu().numpy() for t in pg.find_best(dev(R)))
    ko, tho, sseo, _, gap = po.find_best(R[0])
    assert k[0] == ko or gap / sseo <= TIE_RTOL
    if k[0] == ko:
        assert close(sse[0], sseo, RTOL)[0] and close(th[0], tho, RTOL, scale=np.abs(tho).max())[0]
    pg.close()
