"""CPU check of the algebra behind the cross-Gram path (cwb_set_path 3), independent of
the CUDA code: with the oracle's pool (design Z_k = Zb_k[idx_k], A_k = G_k + lambda_k D) the recurrence

    theta_k <- theta_k - nu A_k^-1 (Z_k^T Z_k*) theta*,
    r^T r   <- r^T r - nu delta* - nu (1 - nu) theta*^T G_k* theta*,   delta_k = 2 theta_k^T s_k - theta_k^T G_k theta_k

run in numpy from theta^[0] = A^-1 Z^T r^[0] alone (the residuals are never updated) selects the same learners as
the oracle's Alg. 1 and reproduces its SSE / risk traces and theta_agg.  This pins the identity the
GPU path implements; the GPU path itself is compared with the oracle in tests/test_gpu_gram.py."""
import numpy as np
import pytest

import cwb_synth as S
from oracle import oracle as O


def gram_recurrence(pool, Y, nu, M):
    K, d, n = pool.K, pool.d, pool.n
    Z = [pool.Zb[k][pool.idx[k]] for k in range(K)]               # n x d designs
    A = [pool.G[k] + pool.lam[k] * pool.D for k in range(K)]
    Ainv = [np.linalg.inv(a) for a in A]
    C = {(k, kp): Z[k].T @ Z[kp] for k in range(K) for kp in range(K)}  # the cross Gram, block by block
    B = Y.shape[0]
    ks_tr = np.zeros((M, B), dtype=np.int64)
    sse_tr = np.zeros((M, B))
    risk_tr = np.zeros((M, B))
    agg = np.zeros((B, K, d))
    for b in range(B):
        r0 = Y[b] - Y[b].mean()
        rr = float(r0 @ r0)
        th = [Ainv[k] @ (Z[k].T @ r0) for k in range(K)]
        for m in range(M):
            s = [A[k] @ th[k] for k in range(K)]
            delta = np.array([2 * th[k] @ s[k] - th[k] @ pool.G[k] @ th[k] for k in range(K)])
            k = int(np.argmax(delta))                               # lowest k on ties (argmax keeps the first)
            t = th[k].copy()
            sse_tr[m, b] = rr - delta[k]
            rr = rr - nu * delta[k] - nu * (1 - nu) * (t @ pool.G[k] @ t)
            risk_tr[m, b] = rr / (2 * n)
            ks_tr[m, b] = k
            agg[b, k] += nu * t
            for kk in range(K):
                th[kk] = th[kk] - nu * Ainv[kk] @ (C[(kk, k)] @ t)
    return ks_tr, sse_tr, risk_tr, agg


@pytest.mark.parametrize("name,reps,M", [("R0", range(8), 100), ("R1", range(6), 120)])
def test_cross_gram_recurrence_reproduces_alg1(name, reps, M):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    pool = O.Pool(ds.X, O.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots),
                  O.MODE_BINNED)
    ref = pool.train(ds.Y, nu=c.nu, M=M)
    ks, sse, risk, agg = gram_recurrence(pool, ds.Y, c.nu, M)
    assert (ks == ref.k_trace).all()
    assert np.allclose(sse, ref.sse_trace, rtol=1e-9, atol=1e-12 * np.abs(ref.sse_trace).max())
    assert np.allclose(risk, ref.risk_trace, rtol=1e-9)
    assert np.allclose(agg, ref.theta_agg, rtol=1e-9, atol=1e-12 * np.abs(ref.theta_agg).max())


def test_cross_gram_block_from_joint_bin_counts():
    """The identity behind the cross-Gram build (k_gram_joint), independent of the CUDA code: rows of one cell
    (l, l') of a pair of binned learners have identical basis rows in both, so
        Z_k^T Z_k' = Zb_k^T C Zb_k',   C[l][l'] = #{i : idx_k(i) = l, idx_k'(i) = l'}
    -- binMatMat's counts-times-design-point-products (G_k = Zb_k^T diag(c) Zb_k) for two index
    vectors; for k' = k, C is diag(bin counts) and the block is G_k."""
    ds = S.make("R1", reps=[0])
    pool = O.Pool(ds.X, O.Config(), O.MODE_BINNED)
    K, ns = pool.K, pool.n_star
    for k in range(K):
        for kp in (k, (k + 1) % K, (k + 3) % K):
            Cn = np.zeros((ns, ns))
            np.add.at(Cn, (pool.idx[k].astype(np.int64), pool.idx[kp].astype(np.int64)), 1.0)
            assert Cn.sum() == pool.n
            blk = pool.Zb[k].T @ Cn @ pool.Zb[kp]
            ref = pool.Zb[k][pool.idx[k]].T @ pool.Zb[kp][pool.idx[kp]]
            assert np.allclose(blk, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
            if kp == k:
                assert np.allclose(blk, pool.G[k], rtol=1e-12, atol=1e-12 * np.abs(ref).max())
