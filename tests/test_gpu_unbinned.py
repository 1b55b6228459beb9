"""GPU parity of the unbinned ("nb") learners (cwb_config.unbinned = 1, csrc/cwb_nb.cu,
SURVEY NEXT-3) against the oracle's unbinned mode (basis at the raw x, dense products,
P:L842-846), on the same seeded inputs.  Agreement rules as tests/parity_util.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, TIE_RTOL, assert_train_parity, cfg_of, close  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(out):
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def gcfg(c):
    return cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                      degree=c.degree, df=c.df, unbinned=1)


@pytest.mark.parametrize("name,reps,M", [("R0", None, None), ("R1", None, None), ("R2", range(0, 1024, 111), 60)])
def test_unbinned_train_matches_oracle(name, reps, M):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    M = M or c.M
    po = O.Pool(ds.X, cfg_of(c), O.MODE_UNBINNED)
    pg = cwb.Pool(dev(ds.X), gcfg(c))
    lam = pg.lam()
    assert np.abs(lam - po.lam).max() <= 1e-9 * np.abs(po.lam).max()   # df -> lambda on G = Z^T Z at x
    g = host(pg.train(dev(ds.Y), nu=c.nu, M=M))
    pg.status()
    o = po.train(ds.Y, nu=c.nu, M=M, threads=8)
    assert_train_parity(g, o, c.n, tag=f"{name} unbinned")
    pg.close()


@pytest.mark.parametrize("name,B", [("R1", 5), ("R2", 2), ("R3", 1)])
def test_unbinned_find_best_matches_oracle(name, B):
    ds = S.make(name, reps=range(B))
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_UNBINNED)
    pg = cwb.Pool(dev(ds.X), gcfg(c))
    R = ds.Y - ds.Y.mean(1, keepdims=True)
    k, th, sse = [t.cpu().numpy() for t in pg.find_best(dev(R))]
    for b in range(B):
        ko, tho, sseo, sall, gap = po.find_best(R[b])
        if k[b] != ko:
            assert gap / sseo <= TIE_RTOL
            continue
        ok, e = close(th[b], tho, RTOL, scale=np.abs(tho).max())
        assert ok, e
        ok, e = close(sse[b], sseo, RTOL)
        assert ok, e
    pg.close()


def test_unbinned_unsupported_calls():
    ds = S.make("R0")
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gcfg(c))
    Y = dev(ds.Y)
    for call in (lambda: pg.train_acwb(Y, M=2), lambda: pg.train_bernoulli(dev((ds.Y > 0).astype(float)), M=2)):
        with pytest.raises(cwb.CwbError) as e:
            call()
        assert e.value.name == "CWB_EUNSUPPORTED"
    pg.close()
    with pytest.raises(cwb.CwbError) as e:
        cwb.Pool(dev(ds.X), cwb.Config(n_star_rule=2, n_star_fixed=21, n_knots=4, degree=2, unbinned=1))
    assert e.value.name == "CWB_EUNSUPPORTED"


def test_unbinned_predict_matches_oracle():
    ds = S.make("R1", reps=range(6))
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_UNBINNED)
    pg = cwb.Pool(dev(ds.X), gcfg(c))
    out = pg.train(dev(ds.Y), nu=c.nu, M=40)
    pg.status()
    off, agg = out["offset"], out["theta_agg"]
    rng = np.random.default_rng(3)
    Xn = ds.X[:, rng.choice(c.n, 300)] + rng.normal(0, 0.5, (c.K, 300))  # includes values outside the range
    g = pg.predict(dev(Xn), off, agg).cpu().numpy()
    o = po.predict(Xn, off.cpu().numpy(), agg.cpu().numpy())
    ok, e = close(g, o, 1e-12, scale=np.abs(o).max())
    assert ok, e
    pg.close()
