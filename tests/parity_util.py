"""Shared helpers of the GPU parity tests: agreement rules.

* idx / bins: bit-exact.
* k* sequences: identical per replication, except at a verified near tie: the
  oracle's best and second-best SSE within TIE_RTOL relative -- then either
  choice is correct and the two runs may legitimately diverge afterwards; the
  comparison of that replication stops at the tie (its remaining iterations
  are checked by invariants only).
* floating point: relative 1e-9 (north_star's agreement tolerance), with an
  absolute floor of 1e-12 of the quantity's scale.
"""
import numpy as np

RTOL = 1e-9
# north_star / SURVEY 8(c) G11: selected-learner sequences are identical except at SSE ties within
# 1e-12 relative (the oracle's best and second-best)
TIE_RTOL = 1e-12


def cfg_of(c):
    from oracle import oracle as O
    return O.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                    degree=c.degree, df=c.df)


def gpu_cfg_of(c):
    from paper_2110_03513_b200 import cwb
    return cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                      degree=c.degree, df=c.df)


def close(a, b, rtol=RTOL, scale=None):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    s = np.abs(b).max() if scale is None else scale
    err = np.abs(a - b)
    ok = err <= rtol * np.maximum(np.abs(b), 1e-3 * s) + 1e-12 * s
    return bool(ok.all()), float((err / np.maximum(np.abs(b), 1e-300)).max()) if a.size else 0.0


def compare_traces(gpu_k, orc_k, orc_gap, orc_sse):
    """Returns (first_divergence[B] (M if none), list of (m, b) verified ties).  The SSE gap is
    measured relative to the best SSE with the agreement rules' absolute floor of 1e-12 of the
    targets' scale ("absolute floor 1e-12 ||y||^2"; the largest SSE of the batch stands
    for ||r||^2): two learners that both fit the residual exactly (SSE ~ 0, e.g. two training rows
    and three coefficients) are a tie whatever rounding noise separates them."""
    M, B = orc_k.shape
    first = np.full(B, M, dtype=np.int64)
    ties = []
    floor = 1e-12 * float(np.abs(orc_sse).max()) if orc_sse.size else 0.0
    for b in range(B):
        bad = np.nonzero(gpu_k[:, b] != orc_k[:, b])[0]
        if len(bad) == 0:
            continue
        m = int(bad[0])
        rel = orc_gap[m, b] / max(abs(orc_sse[m, b]), floor, 1e-300)
        assert rel <= TIE_RTOL, (
            f"replication {b} iteration {m}: gpu k={gpu_k[m, b]} oracle k={orc_k[m, b]} "
            f"but the oracle's SSE gap is {rel:.3e} relative (not a tie)")
        first[b] = m
        ties.append((m, b))
    return first, ties


def assert_train_parity(g, o, n, tag="", min_full=0.9):
    """g: dict of numpy arrays from the GPU; o: oracle TrainResult.  min_full: share of the
    replications that must follow the oracle over all iterations (every divergence is a verified
    tie either way; tiny problems with exact fits may tie on purpose)."""
    M, B = o.k_trace.shape
    first, ties = compare_traces(g["k_trace"], o.k_trace, o.gap_trace, o.sse_trace)
    full = first == M
    assert full.mean() >= min_full, f"{tag}: too many tie divergences {ties}"
    ok, e = close(g["offset"], o.offset, 1e-12)
    assert ok, f"{tag}: offset rel err {e}"
    for b in range(B):
        m = first[b]
        if m == 0:
            continue
        for key, ref in (("sse_trace", o.sse_trace), ("risk_trace", o.risk_trace)):
            ok, e = close(g[key][:m, b], ref[:m, b], RTOL, scale=np.abs(ref[:, b]).max())
            assert ok, f"{tag}: {key} replication {b} rel err {e}"
    if full.any():
        ok, e = close(g["theta_agg"][full], o.theta_agg[full], RTOL, scale=np.abs(o.theta_agg[full]).max())
        assert ok, f"{tag}: theta_agg rel err {e}"
    return first, ties


def follow_parity(g, po, Y, nu, M, tag="", threads=8, report=True):
    """Tie-following comparison: the oracle runs Alg. 1 on the target vectors Y
    (rows = the GPU's replications, in the order of g's columns) and takes the GPU's learner only at a
    verified near tie (its SSE within TIE_RTOL relative of the oracle's minimum); every selected-learner
    index must then match bit for bit and the SSE / risk traces, theta_agg and the offsets agree within
    the tolerances.  g: dict of numpy arrays of exactly these replications.  Returns followed[B] (the
    number of iterations at which the oracle took the GPU's choice at a tie), printed when report."""
    o, followed = po.train_follow(Y, g["k_trace"], tie_rtol=TIE_RTOL, nu=nu, M=M, threads=threads)
    bad = np.argwhere(o.k_trace != g["k_trace"])
    assert len(bad) == 0, f"{tag}: non-tie selections differ at (m, b) = {bad[:5].tolist()}"
    for key, ref in (("sse_trace", o.sse_trace), ("risk_trace", o.risk_trace)):
        ok, e = close(g[key], ref, RTOL, scale=np.abs(ref).max())
        assert ok, f"{tag}: {key} rel err {e}"
    ok, e = close(g["theta_agg"], o.theta_agg, RTOL, scale=np.abs(o.theta_agg).max())
    assert ok, f"{tag}: theta_agg rel err {e}"
    ok, e = close(g["offset"], o.offset, 1e-12)
    assert ok, f"{tag}: offset rel err {e}"
    if report:
        print(f"[parity] {tag}: {g['k_trace'].shape[1]} replications x {M} iterations identical; "
              f"ties followed: {int(followed.sum())} (tie rule {TIE_RTOL:g} relative)")
    return followed
