"""GPU parity of the streaming findBestBaselearner H1 (csrc/cwb_stream.cu: per-chunk
gather plan of the binMatVec sums) against the oracle's Algorithm
binMatVec, and against the other narrow H1 (per-warp MATCH.ANY histograms).

Sizes span one chunk (8192 rows), several chunks with a ragged tail, the full R3/R4
data, 1..4 residual columns (misaligned columns when n is odd), u8 and u16 index
vectors, n* from 2 to 5000 and the fallback above the plan's n* limit.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, TIE_RTOL, cfg_of, close, gpu_cfg_of  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def _check(po, pg, R):
    k, th, sse = [host(t) for t in pg.find_best(dev(R))]
    pg.status()
    for b in range(R.shape[0]):
        ko, tho, sseo, sall, gap = po.find_best(R[b])
        if k[b] != ko:
            assert gap / sseo <= TIE_RTOL, (b, k[b], ko)
            continue
        ok, e = close(th[b], tho, RTOL, scale=np.abs(tho).max())
        assert ok, e
        ok, e = close(sse[b], sseo, RTOL)
        assert ok, e
    return k, th, sse


@pytest.mark.parametrize("name,B", [("R1", 1), ("R2", 1), ("R2", 3), ("R3", 1), ("R4", 1)])
def test_stream_find_best_matches_oracle(name, B):
    ds = S.make(name, reps=range(B))
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    R = ds.Y - ds.Y.mean(1, keepdims=True)
    pg.set_narrow(0)
    k0, th0, sse0 = _check(po, pg, R)
    # the histogram path: same selections, parameters within rounding of each other
    pg.set_narrow(1)
    k1, th1, sse1 = _check(po, pg, R)
    assert (k0 == k1).all()
    assert np.abs(th0 - th1).max() <= 1e-11 * np.abs(th1).max()
    pg.close()


@pytest.mark.parametrize("seed,n,K,ns,B", [(0, 8192, 3, 37, 1), (1, 8193, 4, 256, 2), (2, 24577, 5, 1000, 4),
                                          (3, 16383, 2, 24, 1), (4, 40001, 3, 5000, 3), (5, 9000, 2, 8000, 1),
                                          (6, 300, 7, 17, 1)])
def test_stream_find_best_edge_shapes(seed, n, K, ns, B):
    rng = np.random.default_rng(seed)
    X = np.empty((K, n))
    for k in range(K):
        X[k] = rng.uniform(-3, 7, n) if k % 2 == 0 else rng.standard_normal(n)
    X[0, : n // 3] = X[0, 0]  # a heavy bin (many equal values)
    ocfg = O.Config(n_star_rule=2, n_star_fixed=ns, n_knots=20)
    gcfg = cwb.Config(n_star_rule=2, n_star_fixed=ns, n_knots=20)
    po = O.Pool(X, ocfg, O.MODE_BINNED)
    pg = cwb.Pool(dev(X), gcfg)
    R = rng.standard_normal((B, n))
    pg.set_narrow(0)
    _check(po, pg, R)
    pg.close()


def test_stream_deterministic():
    ds = S.make("R2", reps=range(2))
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(ds.cfg))
    R = dev(ds.Y - ds.Y.mean(1, keepdims=True))
    a = [host(t) for t in pg.find_best(R)]
    b = [host(t) for t in pg.find_best(R)]
    for x, y in zip(a, b):
        assert (x == y).all()
    pg.close()
