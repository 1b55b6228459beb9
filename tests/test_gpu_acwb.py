"""GPU parity of accelerated CWB (Algorithm 2) through the C ABI (cwb_train_acwb)
against the CPU oracle's step-by-step implementation, on the seeded synthetic workloads.
Agreement rules as for CWB (tests/parity_util.py): both learner sequences (k fitted to r,
k_cor fitted to the error-corrected residuals c) identical except after a verified near tie,
floating point within 1e-9 relative."""
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


def first_divergence(g, o, gap, sse):
    """per replication: first iteration where g != o (M if none); asserts it is a verified tie"""
    M, B = o.shape
    first = np.full(B, M)
    for b in range(B):
        bad = np.nonzero(g[:, b] != o[:, b])[0]
        if len(bad):
            m = int(bad[0])
            rel = gap[m, b] / max(abs(sse[m, b]), 1e-300)
            assert rel <= TIE_RTOL, f"replication {b} iteration {m}: gpu {g[m, b]} oracle {o[m, b]}, gap {rel:.2e}"
            first[b] = m
    return first


def check(name, reps, gamma=0.0034, nu=None, M=None, path=0):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    nu = c.nu if nu is None else nu
    M = c.M if M is None else M
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    ro = po.train_acwb(ds.Y, nu=nu, gamma=gamma, M=M, threads=8)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.set_path(path)
    out = pg.train_acwb(dev(ds.Y), nu=nu, gamma=gamma, M=M)
    pg.status()
    g = {k: host(v) for k, v in out.items()}
    f1 = first_divergence(g["k_trace"], ro.k_trace, ro.gap_trace, ro.sse_trace)
    f2 = first_divergence(g["kcor_trace"], ro.kcor_trace, ro.gap_cor_trace, ro.sse_cor_trace)
    first = np.minimum(f1, f2)
    assert (first == M).mean() >= 0.9, f"{name}: too many tie divergences"
    ok, e = close(g["offset"], ro.offset, 1e-12)
    assert ok, e
    for b in range(len(reps)):
        m = first[b]
        if m == 0:
            continue
        for key, ref in (("sse_trace", ro.sse_trace), ("risk_trace", ro.risk_trace)):
            ok, e = close(g[key][:m, b], ref[:m, b], RTOL, scale=np.abs(ref[:, b]).max())
            assert ok, f"{name}: {key} replication {b} rel err {e}"
    full = first == M
    for key, ref in (("theta_f", ro.theta_f), ("theta_h", ro.theta_h)):
        ok, e = close(g[key][full], ref[full], RTOL, scale=max(np.abs(ref[full]).max(), 1e-300))
        assert ok, f"{name}: {key} rel err {e}"
    # the primary model through the aggregated parameters (additivity)
    pred = host(pg.predict(dev(ds.X), dev(g["offset"]), dev(g["theta_f"])))
    ok, e = close(pred[full], ro.f[full], RTOL, scale=np.abs(ro.f).max())
    assert ok, e
    pg.close()
    return g, ro


@pytest.mark.parametrize("path", [1, 2])  # 1: fused kernel (ACC mode), 2: general per-iteration kernels
@pytest.mark.parametrize("name,reps", [("R0", range(8)), ("R1", range(32)), ("R1", range(256)),
                                       ("R2", [0, 1, 2, 3, 700, 1023])])
def test_acwb_parity(name, reps, path):
    if name == "R2" and path == 1:
        pytest.skip("R2 residuals do not fit the ACWB fused kernel (two columns + momentum model)")
    check(name, list(reps), path=path)


def test_acwb_fused_equals_general_and_deterministic():
    ds = S.make("R1", reps=range(64))
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    res = []
    for path in (1, 1, 2):
        pg.set_path(path)
        res.append({k: host(v) for k, v in pg.train_acwb(dev(ds.Y), nu=c.nu, gamma=0.0034, M=c.M).items()})
    for k in res[0]:
        assert (res[0][k] == res[1][k]).all(), k   # run-to-run bitwise (fused)
    assert (res[0]["k_trace"] == res[2]["k_trace"]).all() and (res[0]["kcor_trace"] == res[2]["kcor_trace"]).all()
    for k in ("theta_f", "theta_h"):
        ok, e = close(res[0][k], res[2][k], 1e-11, scale=np.abs(res[2][k]).max())
        assert ok, (k, e)


@pytest.mark.parametrize("path", [1, 2])
def test_acwb_large_momentum_and_step(path):
    check("R1", list(range(8)), gamma=0.5, nu=0.3, M=60, path=path)


def test_acwb_gamma_zero_and_edge_cases():
    g, ro = check("R0", list(range(4)), gamma=0.0)
    assert (g["theta_h"] == 0).all()
    rng = np.random.default_rng(1)
    X = rng.uniform(0, 1, (2, 64))
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=4))
    out = pg.train_acwb(dev(rng.standard_normal((3, 64))), M=0)
    pg.status()
    assert (host(out["theta_f"]) == 0).all() and (host(out["theta_h"]) == 0).all()
    with pytest.raises(cwb.CwbError):
        pg.train_acwb(dev(rng.standard_normal((3, 64))), gamma=-1.0)


@pytest.mark.slow
def test_acwb_r3_sampled():
    check("R3", [0, 1], M=60)


@pytest.mark.parametrize("algo", ["acwb", "bernoulli"])
def test_train_hint_prebuilds_the_plan(algo):
    """cwb_config.train_hint: cwb_init pre-builds the fused plan in the shape of the named training call, which
    then launches only its training kernel; the results are bitwise those of a context built without the hint
    (the plan is a pure function of the pool and the launch shape)."""
    ds = S.make("R1", reps=range(256))
    c = ds.cfg
    Y = S.binary_targets(ds) if algo == "bernoulli" else ds.Y
    outs, nl = [], []
    for hint in (0, 1 if algo == "acwb" else 3):
        gc = gpu_cfg_of(c)
        gc.batch_hint, gc.train_hint = 256, hint
        pg = cwb.Pool(dev(ds.X), gc)
        pg.status()
        l0 = pg.launches()
        if algo == "acwb":
            out = pg.train_acwb(dev(Y), nu=c.nu, gamma=0.0034, M=20)
        else:
            out = pg.train_bernoulli(dev(Y), nu=c.nu, M=20)
        pg.status()
        nl.append(pg.launches() - l0)
        outs.append({k: host(v) for k, v in out.items()})
    assert nl[1] < nl[0], nl  # with the hint: no plan rebuild inside the training call
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k
