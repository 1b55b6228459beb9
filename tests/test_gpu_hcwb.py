"""GPU parity of hybrid CWB (Algorithm 3) through the C ABI (cwb_train_hcwb) against
the CPU oracle: switch iterations, learner sequences (tie-aware), risks and parameters."""
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


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


def first_divergence(g, o, gap, sse):
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


def check(name, reps, nu=None, gamma=0.037, pat0=5, M=None, frac=0.3, path=0):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    nu = c.nu if nu is None else nu
    M = c.M if M is None else M
    vm = S.validation_mask(c.n, frac)
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    ro = po.train_hcwb(ds.Y, vm, nu=nu, gamma=gamma, pat0=pat0, M=M, threads=8)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.set_path(path)
    out = pg.train_hcwb(dev(ds.Y), dev(vm, torch.uint8), nu=nu, gamma=gamma, pat0=pat0, M=M)
    pg.status()
    g = {k: host(v) for k, v in out.items()}
    f1 = first_divergence(g["k_trace"], ro.k_trace, ro.gap_trace, ro.sse_trace)
    kc_o = np.where(ro.kcor_trace < 0, -1, ro.kcor_trace)
    f2 = first_divergence(g["kcor_trace"], kc_o, ro.gap_cor_trace, np.maximum(np.abs(ro.sse_trace), 1e-300))
    first = np.minimum(f1, f2)
    assert (first == M).mean() >= 0.9, f"{name}: too many tie divergences"
    full = first == M
    assert (g["switch_iter"][full] == ro.switch_iter[full]).all()
    ok, e = close(g["offset"], ro.offset, 1e-12)
    assert ok, e
    for b in range(len(reps)):
        m = first[b]
        for key, ref in (("sse_trace", ro.sse_trace), ("risk_trace", ro.risk_trace),
                         ("val_risk_trace", ro.val_risk_trace)):
            ok, e = close(g[key][:m, b], ref[:m, b], RTOL, scale=np.abs(ref[:, b]).max())
            assert ok, f"{name}: {key} replication {b} rel err {e}"
    ok, e = close(g["theta_f"][full], ro.theta_f[full], RTOL, scale=np.abs(ro.theta_f[full]).max())
    assert ok, e
    pred = host(pg.predict(dev(ds.X), dev(g["offset"]), dev(g["theta_f"])))
    ok, e = close(pred[full], ro.f[full], RTOL, scale=np.abs(ro.f).max())
    assert ok, e
    pg.close()
    return g, ro


@pytest.mark.parametrize("path", [1, 2])  # 1: fused persistent kernel (HC mode), 2: per-iteration kernels
@pytest.mark.parametrize("B", [24, 256])  # 256: the bench shape (fused: two 256-thread CTAs per SM)
def test_hcwb_parity_r1_switches(path, B):
    # strong momentum so that replications switch at different iterations inside one launch
    g, ro = check("R1", list(range(B)), nu=0.1, gamma=0.5, pat0=3, M=200, path=path)
    assert (ro.switch_iter < 200).sum() >= B // 2 and len(set(ro.switch_iter.tolist())) > 3


@pytest.mark.parametrize("name,reps,path", [("R0", range(8), 1), ("R0", range(8), 2), ("R1", range(16), 1),
                                            ("R1", range(16), 2), ("R1", range(256), 1), ("R2", [0, 5, 1000], 0)])
def test_hcwb_parity_paper_defaults(name, reps, path):
    check(name, list(reps), path=path)


def test_hcwb_fused_equals_general_all_replications():
    # R1 at its full B = 256: the fused HC kernel and the per-iteration kernels agree
    ds = S.make("R1")
    c = ds.cfg
    vm = dev(S.validation_mask(c.n), torch.uint8)
    res = []
    for path in (1, 2):
        pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
        pg.set_path(path)
        out = pg.train_hcwb(dev(ds.Y), vm, M=c.M)
        pg.status()
        res.append({k: host(v) for k, v in out.items()})
        pg.close()
    a, b = res
    same = (a["k_trace"] == b["k_trace"]).all(0) & (a["switch_iter"] == b["switch_iter"])
    assert same.mean() >= 0.95
    ok, e = close(a["theta_f"][same], b["theta_f"][same], RTOL, scale=np.abs(b["theta_f"]).max())
    assert ok, e
    ok, e = close(a["val_risk_trace"][:, same], b["val_risk_trace"][:, same], RTOL)
    assert ok, e


def test_hcwb_errors():
    rng = np.random.default_rng(0)
    X = rng.uniform(0, 1, (2, 64))
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=4))
    vm = dev(S.validation_mask(64), torch.uint8)
    with pytest.raises(cwb.CwbError):
        pg.train_hcwb(dev(rng.standard_normal((2, 64))), vm, pat0=0)
    with pytest.raises(TypeError):
        pg.train_hcwb(dev(rng.standard_normal((2, 64))), vm.to(torch.int32))
