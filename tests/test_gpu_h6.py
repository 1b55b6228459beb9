"""GPU tests of the general path's residual update H6 (r_i -= nu Zb_k* theta* at idx_k*(i)): the
kernel with the block's zhat columns staged in shared memory (k_h6s, CB = 32 columns per block for
n* <= 640, CB = 16 for n* <= 1280) and the plain k_h6 beyond.  Each shape trains on the general path
against the tie-following oracle; the staged and the plain kernel give bitwise the same
residuals, so the same learner sequences and theta_agg, and r^T r within rounding (partials summed over
other row blocks)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, TIE_RTOL, close  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def data(seed, n, K=3, B=40):
    rng = np.random.default_rng(seed)
    X = np.stack([rng.uniform(-2, 3, n) if k % 2 == 0 else rng.standard_normal(n) for k in range(K)])
    Y = np.stack([np.cos(X[0] * (1 + 0.02 * b)) + 0.5 * X[1] ** 2 * (b % 2) + 0.3 * rng.standard_normal(n)
                  for b in range(B)])
    return X, Y


# n* = 300: CB = 32; 1000: CB = 16; 2000: plain k_h6.  n is not a multiple of the row blocks (ragged tail).
@pytest.mark.parametrize("ns,n", [(300, 30011), (1000, 40003), (2000, 50021)])
def test_general_train_h6_shapes_vs_oracle(ns, n):
    X, Y = data(ns, n)
    M = 30
    pg = cwb.Pool(dev(X), cwb.Config(n_star_rule=2, n_star_fixed=ns, n_knots=20))
    po = O.Pool(X, O.Config(n_star_rule=2, n_star_fixed=ns, n_knots=20), O.MODE_BINNED)
    pg.set_path(2)
    out = pg.train(dev(Y), nu=0.1, M=M)
    pg.status()
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    o, fol = po.train_follow(Y, g["k_trace"], tie_rtol=TIE_RTOL, nu=0.1, M=M, threads=8)
    print(f"[parity] n*={ns} n={n}: ties followed {int(fol.sum())} (tie rule {TIE_RTOL:g})")
    assert (o.k_trace == g["k_trace"]).all()
    for key, ref in (("theta_agg", o.theta_agg), ("sse_trace", o.sse_trace), ("risk_trace", o.risk_trace)):
        ok, e = close(g[key], ref, RTOL, scale=np.abs(ref).max())
        assert ok, f"{key} {e}"
    pg.close()


CODE = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import cwb_synth as S
from parity_util import gpu_cfg_of
from paper_2110_03513_b200 import cwb
ds = S.make(sys.argv[2], reps=range(int(sys.argv[3])))
pg = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), gpu_cfg_of(ds.cfg))
pg.set_path(2)
out = pg.train(torch.as_tensor(ds.Y, device="cuda"), nu=0.05, M=12)
pg.status()
torch.cuda.synchronize()
np.savez(sys.argv[1], **{k: v.cpu().numpy() for k, v in out.items()})
'''


@pytest.mark.parametrize("name,B", [("R2", 96), ("R3", 64), ("R4", 64)])
def test_staged_h6_equals_plain(name, B):
    res = []
    for mode in ("0", "1"):
        path = f"/tmp/h6_{name}_{mode}.npz"
        env = dict(os.environ, CWB_H6=mode, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests")]))
        subprocess.run([sys.executable, "-c", CODE, path, name, str(B)], check=True, env=env, cwd=ROOT)
        res.append(np.load(path))
    a, b = res
    for k in ("k_trace", "theta_agg", "offset"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("sse_trace", "risk_trace"):
        assert np.abs(a[k] - b[k]).max() <= 1e-12 * np.abs(a[k]).max(), k
