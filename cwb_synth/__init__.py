"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: no binning, no P-spline
basis of the learners, no fitting.  It only draws data by the simulation
recipe of the paper's Sec. 4.1.1:

* informative feature j: x_min ~ U[0,100], rho ~ U[0,100], x ~ U[x_min, x_min+rho];
* noise features: N(0, 1);
* effect of feature j: cubic (order 4) spline with 10 inner knots over the
  realised range, coefficients tau_j ~ N(0, 9 I_14) (variance 9, reading G14);
  the simulation basis is scipy.interpolate.BSpline.design_matrix, a library
  routine, so nothing here is shared with the oracle or the CUDA path;
* y = sum_j eta_j + eps, eps ~ N(0, (sd(eta)/SNR)^2) (sd = sample SD, reading G15);
* replication b redraws tau and eps with X fixed (reading G16).

RNG: X from Generator(PCG64(SeedSequence([211003513, cfg]))), replication b
from the b-th child of that SeedSequence's spawn(B).

Configs R0..R4 keep BASELINE.json's size ladder.
The paper's OpenML data sets are not available; these synthetic draws stand
in for them.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 211003513


@dataclass(frozen=True)
class SynthConfig:
    name: str
    n: int
    p_inf: int            # informative features
    p_noise: int          # noise features
    B: int                # replications (target vectors)
    M: int                # boosting iterations
    snr: float
    cfg_id: int
    n_star_rule: int = 0  # learner config travelling with the workload
    n_star_fixed: int = 0
    n_knots: int = 20
    degree: int = 3
    df: float = 5.0
    nu: float = 0.05
    grid_r0: bool = False

    @property
    def K(self) -> int:
        return self.p_inf + self.p_noise


CONFIGS = {
    "R0": SynthConfig("R0", 21, 2, 1, 8, 100, 10.0, 0, n_star_rule=2, n_star_fixed=21,
                      n_knots=4, grid_r0=True),
    "R1": SynthConfig("R1", 1331, 5, 5, 256, 200, 1.0, 1),
    "R2": SynthConfig("R2", 20000, 7, 14, 1024, 200, 1.0, 2),
    "R3": SynthConfig("R3", 200000, 11, 55, 512, 200, 1.0, 3),
    "R4": SynthConfig("R4", 1000000, 42, 42, 64, 200, 1.0, 4),
}


def _sim_knots(lo: float, hi: float, n_inner: int = 10, k: int = 3) -> np.ndarray:
    h = (hi - lo) / (n_inner + 1)
    return lo + h * np.arange(-k, n_inner + 2 + k, dtype=np.float64)


def _sim_basis(x: np.ndarray):
    from scipy.interpolate import BSpline
    lo, hi = float(x.min()), float(x.max())
    t = _sim_knots(lo, hi)
    xc = np.clip(x, t[3], t[-4])
    return BSpline.design_matrix(xc, t, 3)  # sparse n x 14


@dataclass
class Dataset:
    cfg: SynthConfig
    X: np.ndarray                 # K x n (feature-major, float64)
    Y: np.ndarray                 # B_sel x n (replication-major, float64)
    reps: np.ndarray = field(default=None)  # replication ids in Y


def make_X(cfg: SynthConfig) -> tuple[np.ndarray, np.random.SeedSequence]:
    root = np.random.SeedSequence([SEED, cfg.cfg_id])
    g = np.random.Generator(np.random.PCG64(root))
    n, K = cfg.n, cfg.K
    X = np.empty((K, n), dtype=np.float64)
    if cfg.grid_r0:
        # the design points of [-1, 1] by the P:L859 formula itself, lo + (l / (n - 1)) (hi - lo) with the
        # last point set to hi (a linspace grid differs from it by 1 ulp in places)
        grid = -1.0 + (np.arange(n, dtype=np.float64) / float(n - 1)) * 2.0
        grid[-1] = 1.0
        X[0] = grid
        X[1] = grid[g.permutation(n)]
        for j in range(2, K):
            X[j] = g.standard_normal(n)
        return X, root
    for j in range(cfg.p_inf):
        xmin = g.uniform(0.0, 100.0)
        rho = g.uniform(0.0, 100.0)
        X[j] = g.uniform(xmin, xmin + rho, size=n)
    for j in range(cfg.p_inf, K):
        X[j] = g.standard_normal(n)
    return X, root


def make(cfg: SynthConfig | str, reps=None) -> Dataset:
    """X and the target vectors of replications `reps` (default: all B)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    X, root = make_X(cfg)
    reps = np.arange(cfg.B) if reps is None else np.asarray(reps, dtype=np.int64)
    # children are indexed: spawning more than B leaves the first B unchanged
    children = root.spawn(max(cfg.B, int(reps.max()) + 1 if len(reps) else cfg.B))
    n, p = cfg.n, cfg.p_inf
    bases = [_sim_basis(X[j]) for j in range(p)]
    nb = len(reps)
    taus = np.empty((p, 14, nb))
    eps = np.empty((nb, n))
    for c, b in enumerate(reps):
        g = np.random.Generator(np.random.PCG64(children[int(b)]))
        taus[:, :, c] = g.normal(0.0, 3.0, size=(p, 14))
        eps[c] = g.standard_normal(n)
    eta = np.zeros((n, nb))
    for j in range(p):
        eta += bases[j] @ taus[j]
    Y = np.empty((nb, n), dtype=np.float64)
    for c in range(nb):
        e = eta[:, c]
        sd = float(np.std(e, ddof=1))
        Y[c] = e + eps[c] * (sd / cfg.snr)
    return Dataset(cfg, X, Y, reps)


def validation_mask(n: int, frac: float = 0.3, seed: int = 0) -> np.ndarray:
    """Seeded train/validation split for HCWB (30 % validation): uint8[n], 1 = validation row.
    Exactly round(frac * n) validation rows, drawn without replacement."""
    rng = np.random.default_rng(np.random.SeedSequence([SEED, 7, seed]))
    m = np.zeros(n, dtype=np.uint8)
    m[rng.choice(n, size=int(round(frac * n)), replace=False)] = 1
    return m


def binary_targets(ds: Dataset, scale: float = 2.0) -> np.ndarray:
    """Seeded 0/1 targets for the Bernoulli-loss workload (binary classification, the paper's
    real-data setting P:L411): replication c's latent Y[c] standardised to SD `scale` on the
    logit scale, y ~ Bernoulli(1 / (1 + exp(-z))) with uniforms from the replication's own
    seed stream (SeedSequence([SEED, 9, cfg_id, rep]))."""
    out = np.empty_like(ds.Y)
    for c, b in enumerate(ds.reps):
        z = ds.Y[c] - ds.Y[c].mean()
        z = scale * z / z.std(ddof=1)
        u = np.random.default_rng(np.random.SeedSequence([SEED, 9, ds.cfg.cfg_id, int(b)])).uniform(size=z.size)
        out[c] = (u < 1.0 / (1.0 + np.exp(-z))).astype(np.float64)
    return out


def cv_folds(n: int, F: int = 5, seed: int = 0) -> np.ndarray:
    """Seeded assignment of the n rows to F cross-validation folds of (nearly) equal size: uint8[n]."""
    rng = np.random.default_rng(np.random.SeedSequence([SEED, 11, seed]))
    return (rng.permutation(n) % F).astype(np.uint8)
