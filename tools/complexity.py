"""Empirical complexity of one boosting iteration on the GPU ("per-iteration time must be linear in n
and in K", the paper's H4 at P:L1080; its fitted exponents for CWB with binning at P:L460:
M^1.020 K^0.992 (d^2.000 + d^1.005 n*^0.998 + n^0.993)).

Times cwb_train per iteration for an n sweep at fixed K and a K sweep at fixed n (B replications, M iterations,
n* = ceil(sqrt n), d = 24, the paper's simulation recipe of cwb_synth), on the per-iteration kernels (path 2) and on
the persistent fused kernel (path 1) where r fits in shared memory, and fits log t = a + b log x by least squares
over the points.  usage: python tools/complexity.py [B] [M]"""
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
M = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def per_iter_us(n, p_inf, p_noise, path, b=B, reps=3):
    c = dataclasses.replace(S.CONFIGS["R3"], name=f"cx{n}_{p_inf + p_noise}", n=n, p_inf=p_inf,
                            p_noise=p_noise, B=b, M=M, cfg_id=1000 + n % 997 + 7 * (p_inf + p_noise))
    ds = S.make(c)
    X = torch.as_tensor(ds.X, device="cuda")
    Y = torch.as_tensor(ds.Y, device="cuda")
    pool = cwb.Pool(X, cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots))
    pool.set_path(path)
    out = pool.train(Y, nu=c.nu, M=M)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = pool.train(Y, nu=c.nu, M=M, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / M)
    pool.status()
    ns = pool.n_star
    pool.close()
    return min(ts), ns


def fit(xs, ts):
    b, a = np.polyfit(np.log(xs), np.log(ts), 1)
    return b


def sweep(label, xs, fn):
    rows = []
    for x in xs:
        try:
            t, ns = fn(x)
        except Exception as e:  # e.g. the fused kernel does not fit: skip the point
            print(f"  {label}={x:>8d}  skipped: {e}", flush=True)
            continue
        rows.append((x, ns, t))
        print(f"  {label}={x:>8d}  n*={ns:>5d}  {t:10.1f} us/iteration", flush=True)
    xs_, ts_ = np.array([r[0] for r in rows], float), np.array([r[2] for r in rows])
    b = fit(xs_, ts_)
    # a GPU iteration has a fixed part (launch latency, the K-independent H6 in a K sweep): affine fit and
    # t = c0 + c1 x^e
    A = np.vstack([np.ones_like(xs_), xs_]).T
    c = np.linalg.lstsq(A, ts_, rcond=None)[0]
    r2 = 1 - ((ts_ - A @ c) ** 2).sum() / ((ts_ - ts_.mean()) ** 2).sum()
    try:
        from scipy.optimize import curve_fit
        e = curve_fit(lambda x, c0, c1, e: c0 + c1 * x ** e, xs_, ts_, p0=[c[0], c[1], 1.0], maxfev=20000)[0][2]
    except Exception:
        e = float("nan")
    print(f"  log-log exponent of {label}: {b:.3f}; affine t = {c[0]:.1f} + {c[1]:.4g} {label} us (R^2 {r2:.4f}); "
          f"t = c0 + c1 {label}^e: e = {e:.3f}", flush=True)


print(f"# per-iteration time of cwb_train, B = {B}, M = {M}, K = p_inf + p_noise (half informative)")
print("# per-iteration kernels (path 2), K = 32, n sweep")
sweep("n", [25000, 50000, 100000, 200000, 400000, 800000], lambda n: per_iter_us(n, 16, 16, 2))
print("# per-iteration kernels (path 2), n = 200000, K sweep")
sweep("K", [8, 16, 32, 64, 128], lambda k: per_iter_us(200000, k // 2, k - k // 2, 2))
print("# persistent fused kernel (path 1), K = 10, B = 148 (one CTA per SM), n sweep")
sweep("n", [1331, 2662, 5324, 10648, 16000], lambda n: per_iter_us(n, 5, 5, 1, b=148))
print("# persistent fused kernel (path 1), n = 5324, B = 148, K sweep")
sweep("K", [4, 8, 16, 32], lambda k: per_iter_us(5324, k // 2, k - k // 2, 1, b=148))
