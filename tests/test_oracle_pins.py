"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test names the passage (PAPER.md "P:L<n>", SPEC.md "S:L<n>") or the
closed form it checks.  None of them re-types the oracle's formula: they use
worked examples (tests/golden/spec_examples.json), exact rational arithmetic,
closed forms, invariants, independent library routines (scipy BSpline, numpy
dense linear algebra) or brute force.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------- n* rule

@pytest.mark.parametrize("n", [2, 3, 4, 5, 21, 1331, 20000, 200000, 1000000, 99, 100, 101])
def test_n_star_sqrt_is_integer_ceiling(n):
    # P:L859 n* = sqrt(n), rounded up (reading G1): smallest s with s^2 >= n
    s = math.isqrt(n - 1) + 1 if n > 1 else 1
    assert O.n_star(n, 0) == max(s, 2)


@pytest.mark.parametrize("n,expect", [(16, 2), (17, 3), (81, 3), (82, 4), (1000000, 32)])
def test_n_star_fourth_root(n, expect):
    # P:L445 n* = n^(1/4) variant
    assert O.n_star(n, 1) == expect


def test_ladder_bin_counts():
    # SURVEY/BASELINE table: R1 37, R2 142, R3 448, R4 1000
    assert [O.n_star(n) for n in (1331, 20000, 200000, 1000000)] == [37, 142, 448, 1000]


# -------------------------------------------------------------------- bins

def test_build_bins_spec_example():
    g = GOLD["build_bins"]
    z, bnd, idx = O.build_bins(np.array(g["x"], float), g["n_star"])
    assert z.tolist() == g["z"]
    assert idx.tolist() == g["idx"]
    assert bnd.tolist() == [1.0, 3.0]


def test_build_bins_identity_discretisation():
    # x already equal to equally spaced design points -> identity index
    x = np.arange(50, dtype=float) * 3.0 - 7.0
    rng = np.random.default_rng(1)
    perm = rng.permutation(50)
    z, bnd, idx = O.build_bins(x[perm], 50)
    assert (idx == perm).all()
    assert np.abs(z - x).max() <= 1e-12


def _exact_nearest(xs, ns):
    lo, hi = Fraction(min(xs)), Fraction(max(xs))
    zs = [lo + Fraction(l, ns - 1) * (hi - lo) for l in range(ns)]
    out = []
    for x in xs:
        xf = Fraction(x)
        dist = [abs(xf - zz) for zz in zs]
        m = min(dist)
        out.append(dist.index(m))  # tie -> lower bin (P:L861 closed-right intervals)
    return zs, out


@pytest.mark.parametrize("seed,ns", [(0, 7), (1, 2), (2, 13), (3, 37)])
def test_build_bins_brute_force_nearest(seed, ns):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-5, 11, size=200)
    zs, want = _exact_nearest(x.tolist(), ns)
    z, bnd, idx = O.build_bins(x, ns)
    assert idx.tolist() == want
    for a, b in zip(z, zs):  # design points within 1 ulp-ish of the exact grid
        assert abs(Fraction(a) - b) <= Fraction(abs(float(b)) + 1) * Fraction(1, 2**50)
    assert z[-1] == x.max() and z[0] == x.min()


def test_build_bins_ties_go_to_lower_bin():
    # boundary between 0 and 2 is 1, between 2 and 4 is 3 -> lower bin
    z, bnd, idx = O.build_bins(np.array([4.0, 0.0, 1.0, 3.0, 1.0000000000000002]), 3)
    assert idx.tolist() == [2, 0, 0, 1, 1]


@pytest.mark.parametrize("x,ns,err", [([2.0, 2.0, 2.0], 3, "EDEGENERATE"),
                                      ([0.0, 1.0, float("nan")], 3, "ENONFINITE"),
                                      ([0.0, 1.0, 2.0], 1, "EINVAL")])
def test_build_bins_errors(x, ns, err):
    with pytest.raises(O.OracleError) as e:
        O.build_bins(np.array(x), ns)
    assert e.value.name == err


# ------------------------------------------------------------------- basis

def _knots(lo, hi, degree, n_knots):
    h = (hi - lo) / (n_knots + 1)
    return np.array([lo + (q - degree) * h for q in range(n_knots + 2 * degree + 2)])


@pytest.mark.parametrize("degree,n_knots", [(3, 20), (3, 4), (2, 7), (1, 0), (3, 10)])
def test_bspline_matches_scipy(degree, n_knots):
    from scipy.interpolate import BSpline
    lo, hi = -3.25, 17.5
    rng = np.random.default_rng(degree * 100 + n_knots)
    x = np.concatenate([[lo, hi], rng.uniform(lo, hi, 300)])
    B = O.bspline_basis(x, lo, hi, degree, n_knots)
    assert B.shape == (len(x), n_knots + degree + 1)
    t = _knots(lo, hi, degree, n_knots)
    ref = BSpline.design_matrix(x, t, degree, extrapolate=False).toarray()
    assert np.abs(B - ref).max() <= 1e-14
    assert np.abs(B.sum(1) - 1.0).max() <= 1e-14     # partition of unity on [lo, hi]
    assert (B >= -1e-16).all()
    assert ((B > 0).sum(1) <= degree + 1).all()      # local support


def test_uniform_cubic_values_at_knots():
    g = GOLD["uniform_cubic_bspline_at_knot"]["values"]
    B = O.bspline_basis(np.array([0.0, 5.0, 10.0]), 0.0, 10.0, 3, 1)  # knots spacing 5
    # at x = lo the three non-zero cubic B-splines are 1/6, 2/3, 1/6
    nz = B[0][B[0] > 1e-15]
    assert np.allclose(nz, g, rtol=0, atol=1e-15)
    nz_hi = B[2][B[2] > 1e-15]
    assert np.allclose(nz_hi, g, rtol=0, atol=1e-15)


def test_basis_dimension():
    # reading G5: 20 inner knots, degree 3 -> d = 24
    assert O.basis_dim(3, 20) == 24


# ----------------------------------------------------------------- penalty

def test_penalty_d4_spec():
    assert O.penalty(4).tolist() == GOLD["penalty_d4"]["D"]


@pytest.mark.parametrize("d", [5, 8, 24])
def test_penalty_nullspace(d):
    D = O.penalty(d)
    assert np.allclose(D, D.T)
    assert np.abs(D @ np.ones(d)).max() == 0.0
    assert np.abs(D @ np.arange(d, dtype=float)).max() == 0.0
    ev = np.linalg.eigvalsh(D)
    assert (ev > -1e-12).all() and (np.abs(ev) < 1e-10).sum() == 2


# ---------------------------------------------------- binMatMat / binMatVec

def test_bin_mat_mat_spec_examples():
    for g in GOLD["bin_mat_mat"]:
        out = O.bin_mat_mat(np.array(g["Zb"], float), np.array(g["idx"]), np.array(g["w"], float))
        assert out.tolist() == g["out"], g["cite"]


def test_bin_mat_vec_spec_examples():
    for g in GOLD["bin_mat_vec"]:
        out = O.bin_mat_vec(np.array(g["Zb"], float), np.array(g["idx"]), np.array(g["r"], float))
        assert out.tolist() == g["out"], g["cite"]


@pytest.mark.parametrize("seed", range(6))
def test_binned_products_equal_dense_expansion(seed):
    # binned products equal dense products on the expanded Z
    rng = np.random.default_rng(seed)
    n, ns, d = int(rng.integers(5, 2000)), int(rng.integers(2, 60)), int(rng.integers(1, 25))
    Zb = rng.standard_normal((ns, d))
    idx = rng.integers(0, ns, n).astype(np.int32)
    w = rng.uniform(0, 2, n) if seed % 2 else None
    r = rng.standard_normal(n)
    Z = Zb[idx]
    W = np.ones(n) if w is None else w
    ref_mm = Z.T @ (W[:, None] * Z)
    ref_mv = Z.T @ (W * r)
    mm = O.bin_mat_mat(Zb, idx, w)
    mv = O.bin_mat_vec(Zb, idx, r, w)
    scale_mm = np.abs(Z).T @ (W[:, None] * np.abs(Z))
    scale_mv = np.abs(Z).T @ (W * np.abs(r))
    assert (np.abs(mm - ref_mm) <= 1e-12 * scale_mm + 1e-300).all()
    assert (np.abs(mv - ref_mv) <= 1e-12 * scale_mv + 1e-300).all()
    assert np.allclose(O.dense_ztwz(Zb, idx, w), ref_mm, rtol=1e-12, atol=1e-12)
    assert np.allclose(O.dense_ztwr(Zb, idx, r, w), ref_mv, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------- linear algebra

def test_linear_ls_spec():
    g = GOLD["linear_ls"]
    Z = np.array(g["Z"], float)
    r = np.array(g["r"], float)
    th = O.chol_solve(Z.T @ Z, Z.T @ r)
    assert np.allclose(th, g["theta"], rtol=0, atol=1e-13)


def test_cholesky_residual_and_error():
    rng = np.random.default_rng(5)
    A0 = rng.standard_normal((24, 24))
    A = A0 @ A0.T + 24 * np.eye(24)
    L = O.cholesky(A)
    assert np.allclose(np.tril(L), L)
    assert np.abs(L @ L.T - A).max() <= 1e-12 * np.abs(A).max()
    b = rng.standard_normal(24)
    x = O.chol_solve(A, b)
    assert np.abs(A @ x - b).max() <= 1e-10 * (1 + np.abs(b).max())
    with pytest.raises(O.OracleError):
        O.cholesky(-np.eye(3))


# ---------------------------------------------------------------------- df

def test_df_diag_spec():
    g = GOLD["df_diag"]
    G, D = np.array(g["G"], float), np.array(g["D"], float)
    assert abs(O.df(G, D, 1.0, 1) - g["df1_num"] / g["df1_den"]) <= 1e-15
    assert abs(O.df(G, D, 1.0, 2) - g["df2"]) <= 1e-15
    assert abs(O.df(G, D, 0.0, 1) - 2.0) <= 1e-15           # lambda = 0 -> d
    assert O.df(G, D, 1e15, 1) < 1e-14                        # nullity(I) = 0


def test_df_to_lambda_diag_spec():
    g = GOLD["df_to_lambda_diag"]
    lam = O.df_to_lambda(np.array(g["G"], float), np.array(g["D"], float),
                         g["target_num"] / g["target_den"], 1)
    assert abs(lam - g["lambda"]) <= 1e-12


def _hat(Z, D, lam):
    return Z @ np.linalg.solve(Z.T @ Z + lam * D, Z.T)


@pytest.mark.parametrize("seed", range(4))
def test_df_equals_dense_hat_trace(seed):
    # supp. P:L314-318 by explicit n x n hat matrix (numpy), rank-deficient cases included
    rng = np.random.default_rng(seed)
    n, ns = 40, [30, 5, 12, 40][seed]
    x = rng.uniform(0, 1, n)
    z, _, idx = O.build_bins(x, ns)
    Zb = O.bspline_basis(z, z[0], z[-1], 3, 6)
    Z = Zb[idx]
    D = O.penalty(Z.shape[1])
    G = Z.T @ Z
    for lam in [1e-3, 0.7, 13.0, 1e4]:
        H = _hat(Z, D, lam)
        assert abs(O.df(G, D, lam, 1) - np.trace(H)) <= 1e-9
        assert abs(O.df(G, D, lam, 2) - np.trace(2 * H - H @ H)) <= 1e-9
        assert O.df(G, D, lam, 2) >= O.df(G, D, lam, 1) - 1e-12


def test_df_monotone_and_limits():
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 10, 500)
    z, _, idx = O.build_bins(x, 23)
    Zb = O.bspline_basis(z, z[0], z[-1], 3, 20)
    G = O.bin_mat_mat(Zb, idx)
    D = O.penalty(24)
    lams = np.logspace(-6, 9, 40)
    dfs = [O.df(G, D, l, 1) for l in lams]
    assert all(a > b for a, b in zip(dfs, dfs[1:]))
    assert abs(O.df(G, D, 1e-13, 1) - 23.0) < 1e-3            # lambda -> 0: rank(G) = n* = 23 < d
    assert abs(dfs[-1] - 2.0) < 1e-4                          # nullity of D


@pytest.mark.parametrize("kind", [1, 2])
def test_df_to_lambda_calibrates(kind):
    rng = np.random.default_rng(10 + kind)
    x = rng.standard_normal(1331)
    z, _, idx = O.build_bins(x, 37)
    Zb = O.bspline_basis(z, z[0], z[-1], 3, 20)
    G = O.bin_mat_mat(Zb, idx)
    D = O.penalty(24)
    lam = O.df_to_lambda(G, D, 5.0, kind)
    Z = Zb[idx]
    H = _hat(Z, D, lam)
    val = np.trace(H) if kind == 1 else np.trace(2 * H - H @ H)
    assert abs(val - 5.0) <= 1e-8


def test_df_to_lambda_errors():
    G, D = np.diag([2.0, 3.0, 5.0]), O.penalty(3)   # nullity of D = 2
    with pytest.raises(O.OracleError) as e:
        O.df_to_lambda(G, D, 1.5, 1)                 # below nullity
    assert e.value.name == "ECALIB"
    with pytest.raises(O.OracleError):
        O.df_to_lambda(G, D, 3.5, 1)                 # above d


# ------------------------------------------------------------ find best

def _pool(X, **kw):
    return O.Pool(np.asarray(X, float), O.Config(**kw), O.MODE_BINNED)


def test_find_best_singleton():
    rng = np.random.default_rng(0)
    p = _pool(rng.uniform(0, 1, (1, 100)), n_knots=5)
    k, th, sse, sse_all, gap = p.find_best(rng.standard_normal(100))
    assert k == 0 and math.isinf(gap)


def test_find_best_tie_lowest_index():
    rng = np.random.default_rng(1)
    x = rng.uniform(0, 1, 100)
    p = _pool(np.stack([x, x, x]), n_knots=5)
    k, th, sse, sse_all, gap = p.find_best(rng.standard_normal(100))
    assert k == 0 and gap == 0.0 and sse_all[0] == sse_all[1] == sse_all[2]


def test_find_best_orthogonal_residual():
    # r orthogonal to learner A's column space but not B's -> B
    rng = np.random.default_rng(2)
    n = 300
    X = np.stack([rng.uniform(0, 1, n), rng.uniform(0, 1, n)])
    p = _pool(X, n_knots=5)
    ZA = p.Zb[0][p.idx[0]]
    ZB = p.Zb[1][p.idx[1]]
    v = ZB @ rng.standard_normal(p.d)
    r = v - ZA @ np.linalg.lstsq(ZA, v, rcond=None)[0]
    k, th, sse, sse_all, gap = p.find_best(r)
    assert k == 1
    assert abs(sse_all[0] - r @ r) <= 1e-9 * (r @ r)
    assert sse_all[1] < r @ r


@pytest.mark.parametrize("seed", range(5))
def test_find_best_exhaustive(seed):
    # brute force: every learner fitted by numpy dense solve, SSE by full pass
    rng = np.random.default_rng(100 + seed)
    n, K = int(rng.integers(30, 400)), int(rng.integers(1, 7))
    X = rng.uniform(-2, 3, (K, n))
    p = _pool(X, n_knots=int(rng.integers(3, 12)))
    r = rng.standard_normal(n)
    sses, thetas = [], []
    for k in range(K):
        Z = p.Zb[k][p.idx[k]]
        th = np.linalg.solve(Z.T @ Z + p.lam[k] * p.D, Z.T @ r)
        e = r - Z @ th
        sses.append(e @ e)
        thetas.append(th)
        # SSE identity rr - 2 theta^T s + theta^T G theta (exact algebra)
        s = Z.T @ r
        assert abs((r @ r - 2 * th @ s + th @ (Z.T @ Z) @ th) - e @ e) <= 1e-9 * (r @ r)
    k, th, sse, sse_all, gap = p.find_best(r)
    assert k == int(np.argmin(sses))
    assert np.allclose(sse_all, sses, rtol=1e-11, atol=0)
    assert np.allclose(th, thetas[k], rtol=1e-9, atol=1e-12)


def test_pool_df_calibrated_against_dense_hat():
    # every learner of the pool has df1 = 5 by the explicit hat matrix
    rng = np.random.default_rng(7)
    X = np.stack([rng.uniform(0, 50, 400), rng.standard_normal(400), rng.uniform(3, 4, 400)])
    p = _pool(X)
    for k in range(3):
        Z = p.Zb[k][p.idx[k]]
        assert abs(np.trace(_hat(Z, p.D, p.lam[k])) - 5.0) <= 1e-8


# ------------------------------------------------------------------- train

def test_train_linear_m1_spec():
    g = GOLD["train_linear_m1"]
    x = np.array([g["x"]], float)
    p = O.Pool(x, O.Config(n_star_rule=2, n_star_fixed=3, degree=1, n_knots=0, df=2.0), O.MODE_BINNED)
    res = p.train(np.array([g["y"]], float), nu=1.0, M=1)
    assert abs(res.offset[0] - g["offset"]) <= 1e-15
    assert np.allclose(res.f[0], g["f"], rtol=0, atol=1e-13)
    assert abs(res.risk_trace[0, 0] - g["risk"]) <= 1e-25


def test_train_nu_zero_is_offset_only():
    rng = np.random.default_rng(4)
    p = _pool(rng.uniform(0, 1, (3, 200)), n_knots=6)
    y = rng.standard_normal((2, 200))
    res = p.train(y, nu=0.0, M=7)
    assert (res.theta_agg == 0).all()
    assert np.allclose(res.f, y.mean(1, keepdims=True) * np.ones((1, 200)), rtol=0, atol=1e-15)


@pytest.mark.parametrize("nu,M", [(0.05, 60), (0.3, 25), (1.0, 3)])
def test_train_single_learner_closed_form(nu, M):
    # K = 1: r^[m] = (I - nu H)^m r^[0], H = Z (Z^T Z + lambda D)^-1 Z^T (Alg. 1 supp. with K = 1)
    rng = np.random.default_rng(11)
    n = 150
    x = rng.uniform(0, 1, n)
    y = np.sin(6 * x) + 0.3 * rng.standard_normal(n)
    p = _pool(x[None], n_knots=8)
    res = p.train(y[None], nu=nu, M=M)
    Z = p.Zb[0][p.idx[0]]
    H = _hat(Z, p.D, p.lam[0])
    r0 = y - y.mean()
    rM = np.linalg.matrix_power(np.eye(n) - nu * H, M) @ r0
    assert np.abs((y - res.f[0]) - rM).max() <= 1e-11 * np.abs(r0).max()
    # risk trace = (1/n) sum 1/2 r^2 after each update
    rm = r0.copy()
    A = Z.T @ Z + p.lam[0] * p.D
    agg = np.zeros(p.d)
    for m in range(M):
        th = np.linalg.solve(A, Z.T @ rm)
        e = rm - Z @ th
        assert abs(res.sse_trace[m, 0] - e @ e) <= 1e-11 * (r0 @ r0)     # SSE of the fit at m
        agg += nu * th
        rm = rm - nu * H @ rm
        assert abs(res.risk_trace[m, 0] - 0.5 * (rm @ rm) / n) <= 1e-11 * (0.5 * (r0 @ r0) / n)
    assert np.abs(res.theta_agg[0, 0] - agg).max() <= 1e-10 * np.abs(agg).max()   # P:L838 with nu
    assert (res.k_trace == 0).all()


def test_train_invariants_r0():
    import cwb_synth as S
    ds = S.make("R0")
    c = ds.cfg
    cfg = O.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots)
    p = O.Pool(ds.X, cfg, O.MODE_BINNED)
    res = p.train(ds.Y, nu=c.nu, M=c.M, threads=3)
    # train risk non-increasing
    assert (np.diff(res.risk_trace, axis=0) <= 1e-12).all()
    # aggregation: offset + sum_k Z_k theta_agg_k equals the accumulated fit
    pred = p.predict(ds.X, res.offset, res.theta_agg)
    assert np.abs(pred - res.f).max() <= 1e-10 * np.abs(ds.Y).max()
    # SSE_m of the fitted learner never exceeds r^T r before the update: with
    # A = G + lambda D >= G, theta^T G theta <= theta^T s, so SSE <= rr - theta^T s <= rr
    n = ds.cfg.n
    rr_before = np.vstack([0.5 * ((ds.Y - ds.Y.mean(1, keepdims=True)) ** 2).sum(1) / n,
                           res.risk_trace[:-1]]) * 2 * n
    assert (res.sse_trace <= rr_before * (1 + 1e-12)).all()
    # determinism across thread counts
    res1 = p.train(ds.Y, nu=c.nu, M=c.M, threads=1)
    assert (res1.theta_agg == res.theta_agg).all() and (res1.k_trace == res.k_trace).all()


def test_binned_equals_unbinned_on_grid_features():
    # features that coincide with their design points -> identical fits.
    # The grid is built with the design-point expression of P:L859 so x == z exactly.
    n = 41
    lo, hi = -1.0, 1.0
    grid = np.array([lo + (l / (n - 1)) * (hi - lo) for l in range(n)])
    grid[-1] = hi
    rng = np.random.default_rng(9)
    X = np.stack([grid, grid[rng.permutation(n)], grid[rng.permutation(n)]])
    Y = np.stack([np.sin(3 * X[0]) + X[1] ** 2 + 0.1 * rng.standard_normal(n) for _ in range(3)])
    cfg = O.Config(n_star_rule=2, n_star_fixed=n, n_knots=6)
    pb = O.Pool(X, cfg, O.MODE_BINNED)
    pu = O.Pool(X, cfg, O.MODE_UNBINNED)
    assert (pb.idx == np.stack([np.argsort(np.argsort(x)) for x in X])).all()
    rb = pb.train(Y, nu=0.1, M=40)
    ru = pu.train(Y, nu=0.1, M=40)
    assert (rb.k_trace == ru.k_trace).all()
    assert np.allclose(rb.theta_agg, ru.theta_agg, rtol=1e-10, atol=1e-12)


def test_binned_mode_equals_dense_mode():
    # Algorithm binMatVec reaches the dense definition's result
    import cwb_synth as S
    ds = S.make("R1", reps=range(6))
    X = ds.X
    pb = O.Pool(X, O.Config(), O.MODE_BINNED)
    pd = O.Pool(X, O.Config(), O.MODE_DENSE)
    assert np.allclose(pb.lam, pd.lam, rtol=1e-12)
    rb = pb.train(ds.Y, nu=0.05, M=60, threads=6)
    rd = pd.train(ds.Y, nu=0.05, M=60, threads=6)
    assert (rb.k_trace == rd.k_trace).all()
    assert np.allclose(rb.theta_agg, rd.theta_agg, rtol=1e-10, atol=1e-12)
    assert np.allclose(rb.sse_trace, rd.sse_trace, rtol=1e-11)


def test_unbinned_pool_is_penalised_regression_on_x():
    # NEXT-3 basis at x itself: find_best equals numpy penalised LS with g(x)
    rng = np.random.default_rng(13)
    X = rng.uniform(0, 1, (2, 120))
    p = O.Pool(X, O.Config(n_knots=7), O.MODE_UNBINNED)
    r = rng.standard_normal(120)
    k, th, sse, sse_all, gap = p.find_best(r)
    for kk in range(2):
        Z = O.bspline_basis(X[kk], X[kk].min(), X[kk].max(), 3, 7)
        t = np.linalg.solve(Z.T @ Z + p.lam[kk] * p.D, Z.T @ r)
        assert abs(sse_all[kk] - ((r - Z @ t) ** 2).sum()) <= 1e-10 * (r @ r)


# ------------------------------------------------------------------- ACWB (Algorithm 2)

def _acwb_pool(seed=5, K=3, n=300, n_knots=6):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, (K, n))
    y = np.sin(6 * X[0]) + 0.5 * X[min(1, K - 1)] ** 2 + 0.3 * rng.standard_normal(n)
    return O.Pool(X, O.Config(n_knots=n_knots), O.MODE_BINNED), X, y


def _fitted(pool, theta, k):
    return pool.Zb[k][pool.idx[k]] @ theta


def test_acwb_gamma_zero_freezes_momentum_model():
    # gamma = 0 => eta_m = 0 (Alg. 2 line 15) => h^[m] = h^[0] = f^[0] (line 16); theta_h stays 0
    pool, X, y = _acwb_pool()
    r = pool.train_acwb(y[None], nu=0.1, gamma=0.0, M=25)
    assert (r.h == r.offset[0]).all()
    assert (r.theta_h == 0).all()


def test_acwb_first_iteration_is_cwb_first_iteration():
    # theta_1 = 1 => g^[1] = h^[0] = f^[0] (lines 4-5), so r^[1] = y - mean(y) and c^[1] = r^[1] (line 12):
    # the primary and correction learners of iteration 1 equal CWB's first selection
    pool, X, y = _acwb_pool()
    a = pool.train_acwb(y[None], nu=0.1, gamma=0.5, M=1)
    c = pool.train(y[None], nu=0.1, M=1)
    assert a.k_trace[0, 0] == c.k_trace[0, 0] == a.kcor_trace[0, 0]
    assert np.isclose(a.sse_trace[0, 0], c.sse_trace[0, 0], rtol=1e-14)
    assert np.isclose(a.sse_cor_trace[0, 0], c.sse_trace[0, 0], rtol=1e-14)
    # theta_f^[1] = (1-1) 0 + 1 * 0 + nu theta^[1]; theta_h^[1] = eta_1 theta_cor^[1], eta_1 = gamma nu / 1
    k = a.k_trace[0, 0]
    assert np.allclose(a.theta_f[0, k], c.theta_agg[0, k], rtol=1e-13, atol=0)
    assert np.allclose(a.theta_h[0, k], 0.5 * c.theta_agg[0, k], rtol=1e-13, atol=0)


def test_acwb_eta_sequence_read_off_the_oracle():
    # eta_m = gamma nu / vartheta_m with vartheta_m = 2 / (m + 1) (Alg. 2 lines 3 and 15); S:L393's
    # example: gamma = 0.0034, nu = 0.05, m = 3 -> vartheta_3 = 0.5, eta_3 = 3.4e-4.  Read eta off the oracle:
    # one learner on a design-point grid (binned = exact, n* = n) and a LINEAR target: linear functions are in
    # the penalty's null space (D . linear = 0), so the smoother reproduces every residual exactly, the
    # error correction c - b_cor vanishes and theta_cor^[m] = theta^[m], the primary fit of iteration m.  Then
    #   theta_h^[m] - theta_h^[m-1] = eta_m theta^[m],   theta^[m] = (theta_f^[m] - theta_g^[m]) / nu,
    #   theta_g^[m] = (1 - vartheta_m) theta_f^[m-1] + vartheta_m theta_h^[m-1]   (lines 3, 8)
    # from runs of M = m - 1 and M = m iterations.
    n = 41
    x = -1.0 + (np.arange(n) / (n - 1.0)) * 2.0
    x[-1] = 1.0
    y = 3.0 + 2.0 * x
    pool = O.Pool(x[None], O.Config(n_star_rule=2, n_star_fixed=n, n_knots=4), O.MODE_BINNED)
    gamma, nu = 0.0034, 0.05
    runs = [pool.train_acwb(y[None], nu=nu, gamma=gamma, M=M) for M in range(0, 6)]
    for m in range(1, 6):
        a, b = runs[m - 1], runs[m]
        vt = 2.0 / (m + 1)
        th_g = (1.0 - vt) * a.theta_f[0, 0] + vt * a.theta_h[0, 0]
        th = (b.theta_f[0, 0] - th_g) / nu
        dh = b.theta_h[0, 0] - a.theta_h[0, 0]
        j = int(np.argmax(np.abs(th)))
        eta = dh[j] / th[j]
        assert np.allclose(dh, eta * th, rtol=1e-9, atol=1e-12 * np.abs(dh).max()), m
        assert np.isclose(eta, gamma * nu / vt, rtol=1e-9), (m, eta)
        if m == 3:
            assert np.isclose(eta, 3.4e-4, rtol=1e-9)


def test_acwb_aggregation_invariants():
    # the parameters are updated additively, so offset + sum_k Z_k theta_f[k] reproduces the
    # primary model f and offset + sum_k Z_k theta_h[k] the momentum model h
    pool, X, y = _acwb_pool(seed=9, K=4)
    r = pool.train_acwb(y[None], nu=0.05, gamma=0.0034, M=60)
    f = r.offset[0] + sum(_fitted(pool, r.theta_f[0, k], k) for k in range(pool.K))
    h = r.offset[0] + sum(_fitted(pool, r.theta_h[0, k], k) for k in range(pool.K))
    assert np.allclose(f, r.f[0], rtol=0, atol=1e-10 * np.abs(y).max())
    assert np.allclose(h, r.h[0], rtol=0, atol=1e-10 * np.abs(y).max())
    risk = 0.5 * np.mean((y - r.f[0]) ** 2)
    assert np.isclose(risk, r.risk_trace[-1, 0], rtol=1e-12)


def test_acwb_single_learner_matrix_recurrence():
    # With K = 1 findBest always returns learner 0 and its fit is the linear smoother
    # S = Z (Z^T Z + lambda D)^-1 Z^T, so Algorithm 2 becomes a linear recurrence on the fitted
    # vectors; written here with a dense smoother matrix (not the oracle's per-iteration solves).
    pool, X, y = _acwb_pool(seed=2, K=1, n=150)
    Z = pool.Zb[0][pool.idx[0]]
    S = Z @ np.linalg.solve(pool.G[0] + pool.lam[0] * pool.D, Z.T)
    nu, gamma, M = 0.2, 0.3, 40
    f0 = y.mean()
    f = np.full_like(y, f0)
    h = f.copy()
    c = None
    bcor_prev = None
    risks = []
    for m in range(1, M + 1):
        vt = 2.0 / (m + 1)
        g = (1 - vt) * f + vt * h
        rr = y - g
        f = g + nu * (S @ rr)
        c = rr if m == 1 else rr + m / (m + 1) * (c - bcor_prev)
        bcor_prev = S @ c
        h = h + gamma * nu / vt * bcor_prev
        risks.append(0.5 * np.mean((y - f) ** 2))
    r = pool.train_acwb(y[None], nu=nu, gamma=gamma, M=M)
    assert np.allclose(r.f[0], f, rtol=0, atol=1e-10 * np.abs(y).max())
    assert np.allclose(r.h[0], h, rtol=0, atol=1e-10 * np.abs(y).max())
    assert np.allclose(r.risk_trace[:, 0], risks, rtol=1e-9)


def test_acwb_replications_independent_and_threads_deterministic():
    pool, X, y = _acwb_pool(seed=3, K=3)
    rng = np.random.default_rng(0)
    Y = np.stack([y, y[::-1].copy(), rng.standard_normal(y.size)])
    a = pool.train_acwb(Y, nu=0.05, gamma=0.0034, M=30, threads=1)
    b = pool.train_acwb(Y, nu=0.05, gamma=0.0034, M=30, threads=3)
    c = pool.train_acwb(Y[1:2], nu=0.05, gamma=0.0034, M=30)
    for key in ("theta_f", "theta_h", "k_trace", "kcor_trace", "risk_trace"):
        assert (getattr(a, key) == getattr(b, key)).all(), key
    assert (a.theta_f[1] == c.theta_f[0]).all() and (a.k_trace[:, 1] == c.k_trace[:, 0]).all()


# ------------------------------------------------------------------- HCWB (Algorithm 3)

def _hcwb_reference_k1(pool, y, vm, nu, gamma, pat0, M):
    """K = 1: the fits are linear smoothers, S_w = Z (Z^T W Z + lambda D)^-1 Z^T W on the training
    rows before the switch, S = Z (Z^T Z + lambda D)^-1 Z^T on all rows after it."""
    Z = pool.Zb[0][pool.idx[0]]
    w = (vm == 0).astype(float)
    lam, D = pool.lam[0], pool.D
    Sw = Z @ np.linalg.solve(Z.T @ (w[:, None] * Z) + lam * D, (Z * w[:, None]).T)
    S = Z @ np.linalg.solve(Z.T @ Z + lam * D, Z.T)
    f0 = (w * y).sum() / w.sum()
    f = np.full_like(y, f0)
    h = f.copy()
    c = bprev = None
    val = vm == 1
    vprev = 0.5 * np.mean((y[val] - f[val]) ** 2)
    pat, accel, ma, switch = 0, True, 0, M
    vr_trace = []
    for m in range(M):
        if accel:
            ma += 1
            vt = 2.0 / (ma + 1)
            g = (1 - vt) * f + vt * h
            r = y - g
            f = g + nu * (Sw @ r)
            c = r if ma == 1 else r + ma / (ma + 1) * (c - bprev)
            bprev = Sw @ c
            h = h + gamma * nu / vt * bprev
        else:
            f = f + nu * (S @ (y - f))
        vr = 0.5 * np.mean((y[val] - f[val]) ** 2)
        if accel:
            pat = pat + 1 if vr > vprev else 0
            if pat >= pat0:
                accel, switch = False, m + 1
        vprev = vr
        vr_trace.append(vr)
    return f, switch, np.array(vr_trace)


def test_hcwb_single_learner_matches_smoother_formulation():
    pool, X, y = _acwb_pool(seed=4, K=1, n=200)
    rng = np.random.default_rng(7)
    vm = (rng.uniform(size=y.size) < 0.3).astype(np.uint8)
    for nu, gamma, pat0, M in [(0.3, 0.4, 2, 80), (0.1, 0.037, 5, 120), (0.5, 2.0, 1, 40)]:
        f, switch, vr = _hcwb_reference_k1(pool, y, vm, nu, gamma, pat0, M)
        r = pool.train_hcwb(y[None], vm, nu=nu, gamma=gamma, pat0=pat0, M=M)
        assert r.switch_iter[0] == switch
        assert np.allclose(r.f[0], f, rtol=0, atol=1e-9 * np.abs(y).max())
        assert np.allclose(r.val_risk_trace[:, 0], vr, rtol=1e-8)


def test_hcwb_switch_is_one_way_and_aggregation_holds():
    pool, X, y = _acwb_pool(seed=11, K=4, n=400)
    rng = np.random.default_rng(3)
    vm = (rng.uniform(size=y.size) < 0.3).astype(np.uint8)
    r = pool.train_hcwb(y[None], vm, nu=0.3, gamma=1.0, pat0=2, M=150)
    s = r.switch_iter[0]
    assert 0 < s < 150, "expected a switch with strong momentum"
    assert (r.kcor_trace[:s, 0] >= 0).all() and (r.kcor_trace[s:, 0] == -1).all()
    f = r.offset[0] + sum(_fitted(pool, r.theta_f[0, k], k) for k in range(pool.K))
    assert np.allclose(f, r.f[0], rtol=0, atol=1e-10 * np.abs(y).max())
    assert np.isclose(r.offset[0], y[vm == 0].mean(), rtol=1e-14)
    # no switch if the patience is never exhausted
    r2 = pool.train_hcwb(y[None], vm, nu=0.3, gamma=1.0, pat0=10 ** 6, M=40)
    assert r2.switch_iter[0] == 40 and (r2.kcor_trace >= 0).all()


def test_hcwb_errors():
    pool, X, y = _acwb_pool(seed=1, K=2, n=100)
    with pytest.raises(O.OracleError):
        pool.train_hcwb(y[None], np.zeros(y.size, np.uint8))      # no validation rows
    with pytest.raises(O.OracleError):
        pool.train_hcwb(y[None], np.ones(y.size, np.uint8))       # no training rows


# --------------------------------------------------- Bernoulli loss
# Alg. 1 supp. with the Bernoulli loss L(y, f) = log(1 + exp(f)) - y f, y in {0, 1}
# (S:L298-334): pseudo residuals y - sigma(f), offset logit(mean y) (line 2).

def _bern_data(seed=11, K=3, n=400, n_knots=6, df=5.0):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, (K, n))
    eta = 2.0 * np.sin(5 * X[0]) + 1.5 * (X[min(1, K - 1)] - 0.5)
    y = (rng.uniform(size=n) < 1.0 / (1.0 + np.exp(-eta))).astype(float)
    return O.Pool(X, O.Config(n_knots=n_knots, df=df), O.MODE_BINNED), X, y


def test_bernoulli_offset_and_first_iteration():
    p, X, y = _bern_data()
    res = p.train_bernoulli(y, nu=0.1, M=3)
    pb = y.mean()
    assert abs(res.offset[0] - math.log(pb / (1 - pb))) <= 1e-15 * 4     # argmin_c R_emp(c), closed form
    # at f = logit(p) every pseudo residual is y - p: iteration 1 fits the L2 residual y - mean(y)
    k, th, sse, _, _ = p.find_best(y - pb)
    assert res.k_trace[0, 0] == k
    assert abs(res.sse_trace[0, 0] - sse) <= 1e-12 * sse


@pytest.mark.parametrize("frac", [0.5, 0.3])
def test_bernoulli_nu_zero_risk_is_entropy(frac):
    p, X, y = _bern_data()
    n = y.size
    y = np.zeros(n)
    y[: int(frac * n)] = 1.0
    res = p.train_bernoulli(y, nu=0.0, M=4)
    q = y.mean()
    ent = -(q * math.log(q) + (1 - q) * math.log(1 - q))   # log-loss of the constant model; log 2 at q = 1/2
    assert np.abs(res.risk_trace[:, 0] - ent).max() <= 1e-13
    if frac == 0.5:
        assert abs(res.risk_trace[0, 0] - math.log(2.0)) <= 1e-14


def test_bernoulli_single_learner_converges_to_logistic_mle():
    # K = 1: the boosting step theta += nu (G + lambda D)^-1 Z^T (y - sigma(f)) is preconditioned
    # gradient descent on the log-likelihood over span(Z) (which contains the constants:
    # B-splines sum to 1), so its fixed point is the logistic-regression MLE on Z, found here
    # independently by Newton's method (IRLS).
    p, X, y = _bern_data(seed=3, K=1, n=600, n_knots=4, df=7.5)
    res = p.train_bernoulli(y, nu=1.0, M=1500)
    Z = p.Zb[0][p.idx[0]]
    beta = np.zeros(Z.shape[1])
    for _ in range(60):
        eta = Z @ beta
        mu = 1.0 / (1.0 + np.exp(-eta))
        W = mu * (1 - mu)
        beta = beta + np.linalg.solve(Z.T @ (W[:, None] * Z), Z.T @ (y - mu))
    f_mle = Z @ beta
    assert np.abs(res.f[0] - f_mle).max() <= 1e-8 * (1 + np.abs(f_mle).max())
    mu = 1.0 / (1.0 + np.exp(-res.f[0]))
    assert np.abs(Z.T @ (y - mu)).max() <= 1e-9 * y.size             # score equations


def test_bernoulli_risk_decreases_and_aggregation():
    p, X, y = _bern_data(seed=5)
    Y = np.stack([y, 1.0 - y])
    res = p.train_bernoulli(Y, nu=0.05, M=60, threads=2)
    assert (np.diff(res.risk_trace, axis=0) <= 1e-14).all()   # small steps along -gradient
    pred = p.predict(X, res.offset, res.theta_agg)
    assert np.abs(pred - res.f).max() <= 1e-12 * (1 + np.abs(res.f).max())
    # 1 - y is the label swap: f -> -f, same selections
    assert (res.k_trace[:, 0] == res.k_trace[:, 1]).all()
    assert np.abs(res.f[0] + res.f[1]).max() <= 1e-12 * np.abs(res.f).max()
    res1 = p.train_bernoulli(Y, nu=0.05, M=60, threads=1)
    assert (res1.theta_agg == res.theta_agg).all()


def test_bernoulli_binned_mode_equals_dense_mode():
    pb, X, y = _bern_data(seed=8)
    pd = O.Pool(X, O.Config(n_knots=6), O.MODE_DENSE)
    a = pb.train_bernoulli(y, nu=0.1, M=40)
    b = pd.train_bernoulli(y, nu=0.1, M=40)
    assert (a.k_trace == b.k_trace).all()
    assert np.abs(a.theta_agg - b.theta_agg).max() <= 1e-10 * np.abs(b.theta_agg).max()


def test_bernoulli_errors():
    p, X, y = _bern_data()
    with pytest.raises(O.OracleError):
        p.train_bernoulli(np.where(y > 0, 2.0, 0.0), M=2)        # y not in {0, 1}
    with pytest.raises(O.OracleError):
        p.train_bernoulli(np.ones_like(y), M=2)                   # mean(y) = 1


# -------------------------------------------- CV folds: per-replication observation weights (NEXT-4)
# Alg. 1 supp. with 0/1 weights per replication (binMatMat / binMatVec with weights).

def _folds_data(seed=21, K=3, n=360, F=4):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0, 1, (K, n))
    Y = np.stack([np.sin(5 * X[0]) + 0.4 * X[1] + 0.3 * rng.standard_normal(n) for _ in range(F + 1)])
    fold = (rng.permutation(n) % F).astype(np.uint8)
    return O.Pool(X, O.Config(n_knots=6), O.MODE_BINNED), X, Y, fold


def test_folds_without_holdout_equal_plain_cwb():
    p, X, Y, fold = _folds_data()
    res, vr = p.train_folds(Y, fold, 4, np.full(Y.shape[0], -1), nu=0.1, M=30)
    ref = p.train(Y, nu=0.1, M=30)
    assert (res.k_trace == ref.k_trace).all()
    assert np.abs(res.theta_agg - ref.theta_agg).max() <= 1e-12 * np.abs(ref.theta_agg).max()
    assert np.abs(res.risk_trace - ref.risk_trace).max() <= 1e-12 * ref.risk_trace.max()
    assert (vr == 0).all()


def test_folds_held_out_targets_do_not_enter_the_fit():
    p, X, Y, fold = _folds_data()
    reps = np.array([0, 1, 2, 3, 0])
    a, va = p.train_folds(Y, fold, 4, reps, nu=0.1, M=25)
    Y2 = Y.copy()
    for b, f in enumerate(reps):
        Y2[b, fold == f] += 100.0 * (b + 1)  # change only the held-out rows
    b_, vb = p.train_folds(Y2, fold, 4, reps, nu=0.1, M=25)
    assert (a.k_trace == b_.k_trace).all() and (a.theta_agg == b_.theta_agg).all()
    assert (a.offset == b_.offset).all() and (a.sse_trace == b_.sse_trace).all()
    assert (np.abs(vb - va) > 1.0).all()  # the held-out risk sees them


def test_folds_first_fit_is_penalised_weighted_least_squares():
    # iteration 1: theta = (Z^T W Z + lambda D)^-1 Z^T W (y - f0), f0 = training mean; solved here
    # with numpy on the expanded design of the selected learner
    p, X, Y, fold = _folds_data(seed=4)
    res, _ = p.train_folds(Y[:1], fold, 4, np.array([2]), nu=1.0, M=1)
    k = int(res.k_trace[0, 0])
    w = (fold != 2).astype(float)
    y = Y[0]
    f0 = (w * y).sum() / w.sum()
    assert abs(res.offset[0] - f0) <= 1e-13 * abs(f0)
    Z = p.Zb[k][p.idx[k]]
    A = Z.T @ (w[:, None] * Z) + p.lam[k] * O.penalty(p.d)
    th = np.linalg.solve(A, Z.T @ (w * (y - f0)))
    assert np.abs(res.theta_agg[0, k] - th).max() <= 1e-10 * np.abs(th).max()
    sse = (w * (y - f0 - Z @ th) ** 2).sum()
    assert abs(res.sse_trace[0, 0] - sse) <= 1e-10 * sse


def test_folds_risk_traces_match_the_final_fit():
    p, X, Y, fold = _folds_data(seed=9)
    reps = np.array([0, 1, 2, 3, -1])
    res, vr = p.train_folds(Y, fold, 4, reps, nu=0.1, M=15, threads=3)
    for b, f in enumerate(reps):
        w = np.ones(Y.shape[1]) if f < 0 else (fold != f).astype(float)
        e2 = 0.5 * (Y[b] - res.f[b]) ** 2
        assert abs(res.risk_trace[-1, b] - (w * e2).sum() / w.sum()) <= 1e-12 * res.risk_trace[-1, b]
        ho = (1 - w)
        ref = (ho * e2).sum() / ho.sum() if ho.sum() else 0.0
        assert abs(vr[-1, b] - ref) <= 1e-12 * max(ref, 1e-300)
    pred = p.predict(X, res.offset, res.theta_agg)
    assert np.abs(pred - res.f).max() <= 1e-12 * np.abs(res.f).max()


def test_folds_errors():
    p, X, Y, fold = _folds_data()
    with pytest.raises(O.OracleError):
        p.train_folds(Y[:1], fold, 4, np.array([4]), M=2)        # fold id >= F
    with pytest.raises(O.OracleError):
        p.train_folds(Y[:1], np.zeros_like(fold), 1, np.array([0]), M=2)  # fold 0 holds out every row


# ------------------------------------------------------- tie-following mode

def test_follow_own_sequence_is_identity_and_non_ties_are_not_followed():
    p, X, y = _acwb_pool(seed=7)
    Y = np.stack([y, -y, 0.5 * y])
    ref = p.train(Y, nu=0.1, M=40)
    res, fol = p.train_follow(Y, ref.k_trace, tie_rtol=1e-10, nu=0.1, M=40)
    assert (fol == 0).all() and (res.k_trace == ref.k_trace).all() and (res.theta_agg == ref.theta_agg).all()
    # a sequence that differs where the SSE gap is large: not followed, the own choice is kept
    bad = (ref.k_trace + 1) % p.K
    res2, fol2 = p.train_follow(Y, bad, tie_rtol=1e-10, nu=0.1, M=40)
    assert (fol2 == 0).all() and (res2.k_trace == ref.k_trace).all()


def test_follow_takes_a_tie():
    # two identical learners (columns 0 and 1): every selection of learner 0 is an exact tie with 1
    rng = np.random.default_rng(2)
    x = rng.uniform(0, 1, 400)
    X = np.stack([x, x, rng.uniform(0, 1, 400)])
    p = O.Pool(X, O.Config(n_knots=6), O.MODE_BINNED)
    y = np.sin(6 * x) + 0.2 * rng.standard_normal(400)
    ref = p.train(y, nu=0.1, M=20)
    assert (ref.k_trace[:, 0] != 1).all()  # lowest index wins the exact ties
    follow = np.where(ref.k_trace == 0, 1, ref.k_trace)
    res, fol = p.train_follow(y, follow, tie_rtol=0.0, nu=0.1, M=20)
    assert fol[0] == (ref.k_trace == 0).sum() > 0
    assert (res.k_trace == follow).all()
    # the fitted model is the same (learners 0 and 1 are the same function)
    assert np.abs(res.f - ref.f).max() <= 1e-12 * np.abs(ref.f).max()


def test_unbinned_predict_reproduces_the_fit_and_clamps():
    # unbinned pool (basis at x itself): prediction at the training x equals the accumulated fit;
    # values outside [min, max] take the boundary's basis (reading U2)
    rng = np.random.default_rng(12)
    X = rng.uniform(-2, 3, (3, 250))
    y = np.sin(2 * X[0]) + X[1] + 0.2 * rng.standard_normal(250)
    p = O.Pool(X, O.Config(n_knots=6), O.MODE_UNBINNED)
    res = p.train(y, nu=0.2, M=30)
    pred = p.predict(X, res.offset, res.theta_agg)
    assert np.abs(pred - res.f).max() <= 1e-12 * np.abs(res.f).max()
    Xo = X[:, :5].copy()
    Xo[:, 0] = X.min(1) - 10.0
    Xo[:, 1] = X.max(1) + 10.0
    Xc = Xo.copy()
    Xc[:, 0] = X.min(1)
    Xc[:, 1] = X.max(1)
    assert np.abs(p.predict(Xo, res.offset, res.theta_agg) - p.predict(Xc, res.offset, res.theta_agg)).max() == 0.0


def test_no_penalty_learner_calibration():
    # d = 2 (degree 1, no inner knots): Delta has no rows, D = 0, df(lambda) = rank(Z^T Z)
    # = 2 for every lambda: df = 2 is met (any lambda; the oracle reports 1), df = 1.5 is not
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 4, (3, 500))
    p = O.Pool(X, O.Config(n_star_rule=2, n_star_fixed=3, degree=1, n_knots=0, df=2.0), O.MODE_BINNED)
    assert (p.lam == 1.0).all()
    with pytest.raises(O.OracleError) as e:
        O.Pool(X, O.Config(n_star_rule=2, n_star_fixed=3, degree=1, n_knots=0, df=1.5), O.MODE_BINNED)
    assert e.value.name == "ECALIB"


# ------------------------------------------------- n* clamp (reading N1)

def test_n_star_clamped_to_distinct_values():
    # brute force: nsk = min(n*, #distinct), -0.0 and +0.0 one value; rows only in the first nsk bins
    rng = np.random.default_rng(21)
    n = 900  # n* = 30
    X = np.stack([rng.integers(0, 7, n).astype(float),            # 7 distinct
                  rng.choice([-1.5, -0.0, 0.0, 2.25], n),        # 3 distinct (-0 == +0)
                  rng.standard_normal(n),                        # n distinct
                  np.repeat(np.arange(30.0), 30)])               # exactly n* distinct
    p = O.Pool(X, O.Config(n_knots=6, df=2.5), O.MODE_BINNED)  # 3 bins: rank 3, df in (2, 3]
    assert p.n_star == 30
    assert p.nsk.tolist() == [7, 3, 30, 30]
    for k in range(4):
        assert p.idx[k].max() < p.nsk[k]
        # the learner's bins are those of n* = nsk: its design points at the distinct values
        z, bnd = np.empty(p.nsk[k]), np.empty(p.nsk[k] - 1)
        idx = np.empty(n, np.int32)
        O.lib().orc_build_bins(np.ascontiguousarray(X[k]), n, int(p.nsk[k]), z, bnd, idx)
        assert (p.z[k, :p.nsk[k]] == z).all() and (p.idx[k] == idx).all()
        assert (p.z[k, p.nsk[k]:] == p.hi[k]).all()
    # 3 distinct values -> 3 equidistant design points over [-1.5, 2.25]: -1.5, 0.375, 2.25
    assert np.allclose(p.z[1, :3], [-1.5, 0.375, 2.25], rtol=0, atol=1e-15)


def test_clamped_binning_equals_unbinned_on_equidistant_values():
    # with n* = #distinct values, equally spaced, the binned fit equals the unbinned fit.
    # The values are the design points themselves (the P:L859 formula, a linspace differs by
    # 1 ulp); n = 1600 gives n* = 40 > 9 and 13 distinct values, so the clamp decides n*.
    rng = np.random.default_rng(22)
    n = 1600

    def grid(lo, hi, m):
        g = np.array([lo + (l / (m - 1)) * (hi - lo) for l in range(m)])
        g[-1] = hi
        return g
    X = np.stack([rng.choice(grid(-2.0, 3.0, 9), n), rng.choice(grid(0.5, 7.25, 13), n)])
    X[0, :9], X[1, :13] = grid(-2.0, 3.0, 9), grid(0.5, 7.25, 13)  # every value present
    Y = np.stack([np.sin(X[0]) + 0.1 * X[1] ** 2 + 0.2 * rng.standard_normal(n) for _ in range(3)])
    cfg = O.Config(n_knots=4)
    pb = O.Pool(X, cfg, O.MODE_BINNED)
    pu = O.Pool(X, cfg, O.MODE_UNBINNED)
    assert pb.nsk.tolist() == [9, 13]
    assert np.allclose(pb.lam, pu.lam, rtol=1e-9)
    rb = pb.train(Y, nu=0.1, M=50)
    ru = pu.train(Y, nu=0.1, M=50)
    assert (rb.k_trace == ru.k_trace).all()
    assert np.allclose(rb.theta_agg, ru.theta_agg, rtol=1e-9, atol=1e-12)
    assert np.allclose(rb.f, ru.f, rtol=1e-10, atol=1e-12)
