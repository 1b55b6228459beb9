"""GPU parity of CWB with the Bernoulli loss (cwb_train_bernoulli) against the
oracle's Alg. 1 with the same loss (orc_train_loss), on seeded binary targets
(cwb_synth.binary_targets).  Agreement rules as for the L2 loss (tests/parity_util.py)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import assert_train_parity, cfg_of, gpu_cfg_of  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(out):
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("name,reps,M,path", [("R0", None, None, 1), ("R0", None, None, 2), ("R1", None, None, 1),
                                              ("R1", None, None, 2), ("R1", range(37), 60, 1),
                                              ("R2", range(0, 1024, 97), 80, 0)])
def test_bernoulli_matches_oracle(name, reps, M, path):
    # path 1: the persistent kernel (BERN mode), 2: per-iteration kernels
    ds = S.make(name, reps=reps)
    c = ds.cfg
    M = M or c.M
    Y = S.binary_targets(ds)
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.set_path(path)
    g = host(pg.train_bernoulli(dev(Y), nu=c.nu, M=M))
    pg.status()
    o = po.train_bernoulli(Y, nu=c.nu, M=M, threads=8)
    assert_train_parity(g, o, c.n, tag=f"{name} bernoulli")
    pg.close()


@pytest.mark.parametrize("path", [1, 2])
def test_bernoulli_nu_zero_and_m_zero(path):
    ds = S.make("R1", reps=range(3))
    Y = S.binary_targets(ds)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(ds.cfg))
    pg.set_path(path)
    g = host(pg.train_bernoulli(dev(Y), nu=0.0, M=5))
    p = Y.mean(1)
    ent = -(p * np.log(p) + (1 - p) * np.log(1 - p))
    assert np.abs(g["risk_trace"] - ent[None, :]).max() <= 1e-12
    assert np.abs(g["offset"] - np.log(p / (1 - p))).max() <= 1e-13
    assert (g["theta_agg"] == 0).all()
    g0 = host(pg.train_bernoulli(dev(Y), nu=0.05, M=0, traces=False))
    assert np.abs(g0["offset"] - np.log(p / (1 - p))).max() <= 1e-13
    pg.close()


def test_bernoulli_errors_and_determinism():
    ds = S.make("R1", reps=range(4))
    Y = S.binary_targets(ds)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(ds.cfg))
    a = host(pg.train_bernoulli(dev(Y), M=20))
    b = host(pg.train_bernoulli(dev(Y), M=20))
    for k in a:
        assert (a[k] == b[k]).all(), k
    pg.close()
    for (bad, err), path in [(b_, p_) for b_ in ((np.where(Y > 0, 2.0, 0.0), "CWB_EINVAL"),
                                              (np.ones_like(Y), "CWB_EDEGENERATE")) for p_ in (1, 2)]:
        pg = cwb.Pool(dev(ds.X), gpu_cfg_of(ds.cfg))
        pg.set_path(path)
        with pytest.raises(cwb.CwbError) as e:
            pg.train_bernoulli(dev(bad), M=2)
            pg.status()
        assert e.value.name == err
        pg.close()


@pytest.mark.parametrize("path", [1, 2])
def test_bernoulli_skewed_classes(path):
    # class shares 0.3 % .. 99.7 %: |f| up to ~6 at the offset and beyond it as the fit sharpens,
    # so exp(-|f|) spans many binades and sigma saturates (csrc bern_resid, reading B1)
    ds = S.make("R1", reps=range(8))
    c = ds.cfg
    Y = S.binary_targets(ds)
    rng = np.random.default_rng(20211007)
    for b, share in enumerate((0.003, 0.01, 0.05, 0.2, 0.8, 0.95, 0.99, 0.997)):
        y = np.zeros(c.n)
        y[rng.choice(c.n, max(1, int(round(share * c.n))), replace=False)] = 1.0
        Y[b] = y
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.set_path(path)
    g = host(pg.train_bernoulli(dev(Y), nu=0.3, M=60))
    pg.status()
    o = po.train_bernoulli(Y, nu=0.3, M=60, threads=8)
    assert_train_parity(g, o, c.n, tag=f"skewed bernoulli path {path}")
    pg.close()
