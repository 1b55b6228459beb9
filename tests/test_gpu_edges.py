"""Tiny and degenerate shapes on every training entry point and every path (auto, fused,
per-iteration), against the oracle: n down to 2, K = 1, no-penalty learners (d = 2), degree 1-3,
B not a multiple of 32.  Where the oracle rejects a configuration (HCWB with a single training row:
singular training-row G), the GPU must reject it with the same status."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import TIE_RTOL, assert_train_parity  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"
CASES = [  # (n, K, B, n*, degree, knots, df)
    (2, 1, 1, 2, 1, 0, 2.0), (3, 1, 2, 3, 1, 0, 2.0), (5, 2, 3, 5, 1, 1, 2.5), (40, 1, 1, 6, 2, 2, 3.0),
    (300, 1, 1, 17, 3, 4, 4.0), (1000, 2, 1, 30, 3, 20, 5.0), (64, 3, 33, 8, 3, 3, 4.0)]


def dev(a, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=DEV)


def host(out):
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("n,K,B,ns,dg,nk,df", CASES)
@pytest.mark.parametrize("path", [0, 1, 2])
def test_edge_shapes_all_entry_points(n, K, B, ns, dg, nk, df, path):
    rng = np.random.default_rng(n + K + B)
    X = rng.uniform(-1, 2, (K, n))
    Y = np.sin(2 * X[0])[None, :] + 0.3 * rng.standard_normal((B, n))
    Yb = (Y > np.median(Y)).astype(float)
    Yb[:, 0], Yb[:, -1] = 0.0, 1.0  # both classes present
    ocfg = O.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df)
    gcfg = cwb.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df)
    po = O.Pool(X, ocfg, O.MODE_BINNED)

    def pool():
        pg = cwb.Pool(dev(X), gcfg)
        pg.set_path(path)
        return pg

    pg = pool()
    g = host(pg.train(dev(Y), nu=0.2, M=12))
    pg.status()
    assert_train_parity(g, po.train(Y, nu=0.2, M=12), n, tag="train")
    R = Y[:1] - Y[:1].mean()
    k, th, sse = (t.cpu().numpy() for t in pg.find_best(dev(R)))
    ko, tho, sseo, _, gap = po.find_best(R[0])
    assert k[0] == ko or gap <= TIE_RTOL * sseo
    pg.close()

    pg = pool()
    g = host(pg.train_bernoulli(dev(Yb), nu=0.2, M=12))
    pg.status()
    assert_train_parity(g, po.train_bernoulli(Yb, nu=0.2, M=12), n, tag="bernoulli")
    pg.close()

    pg = pool()
    a = host(pg.train_acwb(dev(Y), nu=0.2, gamma=0.01, M=12))
    pg.status()
    assert np.isfinite(a["risk_trace"]).all()
    pg.close()

    vm = S.validation_mask(n)
    try:
        po.train_hcwb(Y, vm, nu=0.2, gamma=0.05, pat0=2, M=12)
        oracle_err = None
    except O.OracleError as e:
        oracle_err = e.name
    pg = pool()
    if oracle_err is None:
        h = host(pg.train_hcwb(dev(Y), dev(vm, torch.uint8), nu=0.2, gamma=0.05, pat0=2, M=12))
        pg.status()
        assert np.isfinite(h["risk_trace"]).all()
    else:
        with pytest.raises(cwb.CwbError) as e:
            pg.train_hcwb(dev(Y), dev(vm, torch.uint8), nu=0.2, gamma=0.05, pat0=2, M=12)
            pg.status()
        # a forced fused path may refuse the shape first (EUNSUPPORTED) -- never accept it
        assert e.value.name == "CWB_" + oracle_err or (path == 1 and e.value.name == "CWB_EUNSUPPORTED")
    pg.close()


@pytest.mark.parametrize("n,K,B,ns,dg,nk,df", CASES)
def test_edge_shapes_folds_and_unbinned(n, K, B, ns, dg, nk, df):
    rng = np.random.default_rng(n + K + B + 1)
    X = rng.uniform(-1, 2, (K, n))
    Y = np.cos(2 * X[0])[None, :] + 0.3 * rng.standard_normal((B, n))
    ocfg = O.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df)
    gcfg = cwb.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df)
    po = O.Pool(X, ocfg, O.MODE_BINNED)
    # CV folds (F = 2): replications cycle through no hold-out, fold 0, fold 1
    F = 2
    fold = S.cv_folds(n, F)
    frep = (np.arange(B) % (F + 1) - 1).astype(np.int32)
    try:
        o, ov = po.train_folds(Y, fold, F, frep, nu=0.2, M=10)
        oracle_err = None
    except O.OracleError as e:
        oracle_err = e.name
    pg = cwb.Pool(dev(X), gcfg)
    if oracle_err is None:
        g = host(pg.train_folds(dev(Y), dev(fold, torch.uint8), F, dev(frep, torch.int32), nu=0.2, M=10))
        pg.status()
        assert_train_parity(g, o, n, tag="folds", min_full=0.0)  # 2 training rows: exact fits tie
    else:
        with pytest.raises(cwb.CwbError) as e:
            pg.train_folds(dev(Y), dev(fold, torch.uint8), F, dev(frep, torch.int32), nu=0.2, M=10)
            pg.status()
        assert e.value.name == "CWB_" + oracle_err
    pg.close()
    if dg != 3:
        return  # unbinned learners are cubic (include/cwb.h)
    pu = O.Pool(X, ocfg, O.MODE_UNBINNED)
    gu = cwb.Config(n_star_rule=2, n_star_fixed=ns, degree=dg, n_knots=nk, df=df, unbinned=1)
    pg = cwb.Pool(dev(X), gu)
    g = host(pg.train(dev(Y), nu=0.2, M=10))
    pg.status()
    assert_train_parity(g, pu.train(Y, nu=0.2, M=10), n, tag="unbinned")
    pg.close()
