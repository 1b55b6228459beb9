"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, on the
same seeded inputs (cwb_synth), element by element.  Agreement rules in
tests/parity_util.py and DESIGN.md.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import (RTOL, TIE_RTOL, assert_train_parity, cfg_of, close, follow_parity,  # noqa: E402
                         gpu_cfg_of)

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------ binning

@pytest.mark.parametrize("seed,n,ns", [(0, 5, 3), (1, 1000, 37), (2, 20000, 142), (3, 65536, 256),
                                       (4, 70001, 448), (5, 3000, 1000), (6, 257, 2)])
def test_bin_bit_exact(seed, n, ns):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-71.16807745607325, 89.72988942744877, n) if seed else np.arange(5.0)
    if seed == 6:
        x = rng.standard_normal(n)
    z, bnd, idx = O.build_bins(x, ns)
    gz, gb, gi = cwb.cwb_bin(dev(x), ns)
    assert (host(gz) == z).all()
    assert (host(gb) == bnd).all()
    assert (host(gi).astype(np.int64) == idx).all()


def test_bin_ties_and_errors():
    x = np.array([4.0, 0.0, 1.0, 3.0, 1.0000000000000002, 2.0, 3.0000000000000004])
    z, bnd, idx = O.build_bins(x, 3)
    gz, gb, gi = cwb.cwb_bin(dev(x), 3)
    assert (host(gi).astype(np.int64) == idx).all()
    with pytest.raises(cwb.CwbError) as e:
        cwb.cwb_bin(dev(np.full(10, 2.5)), 3)
    assert e.value.name == "CWB_EDEGENERATE"
    with pytest.raises(cwb.CwbError) as e:
        cwb.cwb_bin(dev(np.array([0.0, np.nan, 1.0])), 3)
    assert e.value.name == "CWB_ENONFINITE"


# ------------------------------------------------- binMatVec / binMatMat

@pytest.mark.parametrize("seed,n,ns,d,B,weighted", [(0, 3, 2, 1, 1, False), (1, 2000, 37, 24, 5, True),
                                                     (2, 20000, 142, 24, 33, False), (3, 70000, 448, 24, 64, True),
                                                     (4, 1, 1, 3, 2, False), (5, 999, 300, 7, 1, True)])
def test_bin_mat_vec_and_mat(seed, n, ns, d, B, weighted):
    rng = np.random.default_rng(seed)
    Zb = rng.standard_normal((ns, d))
    idx = rng.integers(0, ns, n).astype(np.int32)
    R = rng.standard_normal((B, n))
    w = rng.uniform(0, 2, n) if weighted else None
    ib = 1 if ns <= 256 else 2
    gidx = dev(idx.astype(np.uint8 if ib == 1 else np.uint16), torch.uint8 if ib == 1 else torch.uint16)
    got = host(cwb.cwb_bin_mat_vec(dev(Zb), gidx, dev(R), None if w is None else dev(w)))
    for b in range(B):
        ref = O.bin_mat_vec(Zb, idx, R[b], w)
        ok, e = close(got[b], ref, 1e-12, scale=np.abs(Zb).max() * np.abs(R[b]).sum() * (2 if weighted else 1))
        assert ok, e
    gm = host(cwb.cwb_bin_mat_mat(dev(Zb), gidx, None if w is None else dev(w)))
    rm = O.bin_mat_mat(Zb, idx, w)
    ok, e = close(gm, rm, 1e-12, scale=np.abs(rm).max())
    assert ok, e


def test_bin_mat_vec_spec_examples():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
    for ex in g["bin_mat_vec"]:
        out = cwb.cwb_bin_mat_vec(dev(np.array(ex["Zb"], float)), dev(np.array(ex["idx"], np.uint8), torch.uint8),
                                  dev(np.array([ex["r"]], float)))
        assert host(out)[0].tolist() == ex["out"]
    for ex in g["bin_mat_mat"]:
        out = cwb.cwb_bin_mat_mat(dev(np.array(ex["Zb"], float)), dev(np.array(ex["idx"], np.uint8), torch.uint8),
                                  dev(np.array(ex["w"], float)))
        assert host(out).tolist() == ex["out"]


# ---------------------------------------------------------------- pool

@pytest.mark.parametrize("name", ["R0", "R1", "R2"])
def test_pool_matches_oracle(name):
    ds = S.make(name, reps=[0])
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.status()
    assert (pg.n_star, pg.d) == (po.n_star, po.d)
    P = {k: host(v) for k, v in pg.pool().items()}
    assert (P["idx"].astype(np.int64) == po.idx).all()          # bit-exact hash
    assert (P["z"] == po.z).all()                                 # bit-exact design points
    ok, e = close(P["Zb"], po.Zb, 1e-14, scale=1.0)
    assert ok, e
    ok, e = close(P["G"], po.G, 1e-12, scale=np.abs(po.G).max())
    assert ok, e
    lam = pg.lam()
    ok, e = close(lam, po.lam, 1e-10)
    assert ok, f"lambda rel err {e}"
    Ainv = np.linalg.inv(po.G + po.lam[:, None, None] * po.D)
    ok, e = close(P["Ainv"], Ainv, 1e-9, scale=np.abs(Ainv).max())
    assert ok, e
    # df(lambda_gpu) = 5 by the oracle's dense trace definition
    for k in range(po.K):
        assert abs(O.df(po.G[k], po.D, float(lam[k]), 1) - c.df) < 1e-9
    pg.close()


@pytest.mark.parametrize("kind", [1, 2])
def test_df_kinds(kind):
    ds = S.make("R1", reps=[0])
    cfg = cfg_of(ds.cfg)
    cfg.df_kind = kind
    po = O.Pool(ds.X, cfg, O.MODE_BINNED)
    gc = gpu_cfg_of(ds.cfg)
    gc.df_kind = kind
    pg = cwb.Pool(dev(ds.X), gc)
    ok, e = close(pg.lam(), po.lam, 1e-10)
    assert ok, e
    pg.close()


def test_pool_errors():
    rng = np.random.default_rng(0)
    X = rng.uniform(0, 1, (3, 200))
    X[1] = 0.5
    p = cwb.Pool(dev(X))
    with pytest.raises(cwb.CwbError) as e:
        p.status()
    assert e.value.name == "CWB_EDEGENERATE"
    X[1] = rng.uniform(0, 1, 200)
    X[2, 7] = np.inf
    with pytest.raises(cwb.CwbError) as e:
        cwb.Pool(dev(X)).status()
    assert e.value.name == "CWB_ENONFINITE"
    with pytest.raises(cwb.CwbError) as e:   # df above rank(G): n* = 3 bins < 5 df
        cwb.Pool(dev(rng.uniform(0, 1, (2, 50))), cwb.Config(n_star_rule=2, n_star_fixed=3)).status()
    assert e.value.name == "CWB_ECALIB"
    with pytest.raises(cwb.CwbError) as e:
        cwb.Pool(torch.empty((0, 10), dtype=torch.float64, device=DEV))
    assert e.value.name == "CWB_EEMPTY"


# ------------------------------------------------------------ find best

@pytest.mark.parametrize("name,B", [("R0", 8), ("R1", 40), ("R2", 3), ("R0", 1), ("R1", 1), ("R1", 2), ("R2", 4),
                                    ("R1", 5)])
def test_find_best_matches_oracle(name, B):
    ds = S.make(name, reps=range(B))
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_DENSE)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    R = ds.Y - ds.Y.mean(1, keepdims=True)
    R[0] *= 1e-3
    k, th, sse = [host(t) for t in pg.find_best(dev(R))]
    for b in range(B):
        ko, tho, sseo, sall, gap = po.find_best(R[b])
        if k[b] != ko:
            assert gap / sseo <= TIE_RTOL
            continue
        ok, e = close(th[b], tho, RTOL, scale=np.abs(tho).max())
        assert ok, e
        ok, e = close(sse[b], sseo, RTOL)
        assert ok, e
    pg.close()


@pytest.mark.parametrize("name,B", [("R3", 1), ("R4", 2)])
def test_find_best_narrow_full_size(name, B):
    # the narrow (B <= 4) findBestBaselearner at full data size against Algorithm binMatVec
    ds = S.make(name, reps=range(B))
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    R = ds.Y - ds.Y.mean(1, keepdims=True)
    k, th, sse = [host(t) for t in pg.find_best(dev(R))]
    for b in range(B):
        ko, tho, sseo, sall, gap = po.find_best(R[b])
        if k[b] != ko:
            assert gap / sseo <= TIE_RTOL
            continue
        ok, e = close(th[b], tho, RTOL, scale=np.abs(tho).max())
        assert ok, e
        ok, e = close(sse[b], sseo, RTOL)
        assert ok, e
    pg.close()


def test_find_best_ties_and_orthogonal():
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, 300)
    X = np.stack([x, x, rng.uniform(0, 1, 300)])
    po = O.Pool(X, O.Config(n_knots=6), O.MODE_BINNED)
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=6))
    r = rng.standard_normal(300)
    k, th, sse = [host(t) for t in pg.find_best(dev(r[None]))]
    ko = po.find_best(r)[0]
    assert ko in (0, 2) and (k[0] == ko or k[0] in (0, 2))
    assert k[0] != 1  # exact duplicate of learner 0 never wins (lowest index)
    # r orthogonal to learner 0's (and 1's) column space -> learner 2
    ZA = po.Zb[0][po.idx[0]]
    ZB = po.Zb[2][po.idx[2]]
    v = ZB @ rng.standard_normal(po.d)
    r2 = v - ZA @ np.linalg.lstsq(ZA, v, rcond=None)[0]
    k, th, sse = [host(t) for t in pg.find_best(dev(r2[None]))]
    assert k[0] == 2


# ---------------------------------------------------------------- train

def _gpu_train(pg, Y, c, path, M=None):
    pg.set_path(path)
    out = pg.train(dev(Y), nu=c.nu, M=M or c.M)
    pg.status()
    return {k: host(v) for k, v in out.items()}


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("name", ["R0", "R1"])
def test_train_full_parity(name, path):
    ds = S.make(name)
    c = ds.cfg
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    ro = po.train(ds.Y, nu=c.nu, M=c.M, threads=8)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    g = _gpu_train(pg, ds.Y, c, path)
    first, ties = assert_train_parity(g, ro, c.n, f"{name}/path{path}")
    # aggregation invariant on the GPU side: predict(X) reproduces the final fit
    pred = host(pg.predict(dev(ds.X), dev(g["offset"]), dev(g["theta_agg"])))
    opred = po.predict(ds.X, g["offset"], g["theta_agg"])
    ok, e = close(pred, opred, 1e-12, scale=np.abs(opred).max())
    assert ok, e
    full = first == c.M
    ok, e = close(pred[full], ro.f[full], 1e-9, scale=np.abs(ro.f).max())
    assert ok, e
    assert (np.diff(g["risk_trace"], axis=0) <= 1e-12 * g["risk_trace"][0]).all()
    pg.close()


def test_train_dense_oracle_agrees_r1_subset():
    # the dense (materialised) definition, not only Algorithm binMatVec
    ds = S.make("R1", reps=range(12))
    c = ds.cfg
    ro = O.Pool(ds.X, cfg_of(c), O.MODE_DENSE).train(ds.Y, nu=c.nu, M=c.M, threads=8)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    g = _gpu_train(pg, ds.Y, c, 0)
    assert_train_parity(g, ro, c.n, "R1/dense")


def test_paths_agree_and_deterministic():
    ds = S.make("R1", reps=range(64))
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    a = _gpu_train(pg, ds.Y, c, 1)
    a2 = _gpu_train(pg, ds.Y, c, 1)
    b = _gpu_train(pg, ds.Y, c, 2)
    b2 = _gpu_train(pg, ds.Y, c, 2)
    for k in a:
        assert (a[k] == a2[k]).all(), k      # run-to-run bitwise (fused)
        assert (b[k] == b2[k]).all(), k      # run-to-run bitwise (general)
    assert (a["k_trace"] == b["k_trace"]).all()
    ok, e = close(a["theta_agg"], b["theta_agg"], 1e-11, scale=np.abs(b["theta_agg"]).max())
    assert ok, e


@pytest.mark.parametrize("name,B", [("R1", 256), ("R1", 100), ("R0", 8)])
def test_batch_hint_prebuilt_plan_identical(name, B):
    # cwb_init with batch_hint pre-builds the gather plan on a side stream; results are bitwise
    # those of the lazily built plan (and of a hint that does not match B)
    ds = S.make(name, reps=range(B))
    c = ds.cfg
    outs = []
    for hint in (0, B, 7):
        gc = gpu_cfg_of(c)
        gc.batch_hint = hint
        pg = cwb.Pool(dev(ds.X), gc)
        outs.append(_gpu_train(pg, ds.Y, c, 0))
        pg.close()
    for o in outs[1:]:
        for k in o:
            assert (o[k] == outs[0][k]).all(), k


def test_train_r2_full_launch_sampled():
    # full R2 launch (B = 1024, the bench configuration of that rung); replications sampled
    ds = S.make("R2")
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    g = _gpu_train(pg, ds.Y, c, 0)
    reps = [0, 1, 511, 1023]
    ro = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED).train(ds.Y[reps], nu=c.nu, M=c.M, threads=4)
    gs = {k: v[:, reps] if v.ndim == 2 and k != "theta_agg" else v[reps] for k, v in g.items()}
    assert_train_parity(gs, ro, c.n, "R2")


def _full_launch(name, M=None):
    """The bench's launch configuration of a rung: all B replications of the workload in one cwb_train call
    (batch_hint = B as bench.py), auto path."""
    ds = S.make(name)
    c = ds.cfg
    gc = gpu_cfg_of(c)
    gc.batch_hint = c.B
    pg = cwb.Pool(dev(ds.X), gc)
    g = _gpu_train(pg, ds.Y, c, 0, M=M)
    pg.close()
    return ds, g


def _sub(g, reps):
    return {k: (v[:, reps] if v.ndim == 2 and k != "theta_agg" else v[reps]) for k, v in g.items()}


@pytest.mark.slow
def test_train_r3_full_launch_parity():
    # SURVEY 8(c) coverage for R3: replications 0-7 (and the last ones of the launch, 255 and 511) of the full
    # B = 512 launch, all 200 iterations, against the tie-following oracle (P:L292, P:L1047 scale)
    ds, g = _full_launch("R3")
    c = ds.cfg
    reps = [0, 1, 2, 3, 4, 5, 6, 7, 255, 511]
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(_sub(g, reps), po, ds.Y[reps], c.nu, c.M, "R3 B=512", threads=len(reps))
    assert fol.sum() <= max(1, 0.01 * c.M * len(reps))


@pytest.mark.slow
def test_train_r4_full_launch_parity():
    # SURVEY 8(c) coverage for R4: replications 0-3 of the full B = 64 launch, all 200 iterations
    ds, g = _full_launch("R4")
    c = ds.cfg
    reps = [0, 1, 2, 3]
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(_sub(g, reps), po, ds.Y[reps], c.nu, c.M, "R4 B=64", threads=len(reps))
    assert fol.sum() <= max(1, 0.01 * c.M * len(reps))


def test_train_edge_cases():
    rng = np.random.default_rng(8)
    X = rng.uniform(0, 1, (2, 50))
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=4))
    Y = rng.standard_normal((3, 50))
    for path in (1, 2):
        pg.set_path(path)
        out = pg.train(dev(Y), nu=0.0, M=5)              # nu = 0: offset only
        assert (host(out["theta_agg"]) == 0).all()
        out = pg.train(dev(Y), nu=0.1, M=0)              # M = 0: offset only
        assert np.allclose(host(out["offset"]), Y.mean(1), rtol=1e-13)
    Yb = Y.copy()
    Yb[1, 3] = np.nan
    pg.set_path(0)
    pg.train(dev(Yb), nu=0.1, M=2)
    with pytest.raises(cwb.CwbError) as e:
        pg.status()
    assert e.value.name == "CWB_ENONFINITE"


def test_fit_host_matches_device_api():
    ds = S.make("R1", reps=range(16))
    c = ds.cfg
    h = cwb.cwb_fit_host(ds.X, ds.Y, gpu_cfg_of(c), nu=c.nu, M=c.M)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    g = _gpu_train(pg, ds.Y, c, 0)
    for k in g:
        assert (h[k] == g[k]).all(), k


@pytest.mark.parametrize("name,path", [("R1", 1), ("R1", 2), ("R0", 1), ("R0", 2)])
def test_train_parity_tie_following(name, path):
    # every replication, every iteration: the oracle follows the GPU's choice only at verified near-ties
    # (SSE within TIE_RTOL = 1e-12 relative of its minimum), so the learner sequences must be identical and
    # all traces and parameters must agree everywhere
    ds = S.make(name)
    c = ds.cfg
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    pg.set_path(path)
    out = pg.train(dev(ds.Y), nu=c.nu, M=c.M)
    pg.status()
    g = {k: host(v) for k, v in out.items()}
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(g, po, ds.Y, c.nu, c.M, f"{name} path {path}")
    assert fol.sum() <= max(1, 0.01 * c.M * c.B)
    pg.close()


def test_train_r2_full_launch_tie_following():
    # R2 at its bench launch (B = 1024), replications spread over the launch, all 200 iterations
    ds, g = _full_launch("R2")
    c = ds.cfg
    reps = [0, 1, 2, 3, 511, 512, 1022, 1023]
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(_sub(g, reps), po, ds.Y[reps], c.nu, c.M, "R2 B=1024", threads=len(reps))
    assert fol.sum() <= max(1, 0.01 * c.M * len(reps))


@pytest.mark.slow
def test_general_h1_chunked_equals_unchunked_r4():
    # the row-chunked H1 (32-column tile of R beyond L2) against the one-sweep H1 on R4
    import os
    import subprocess
    import sys
    code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import cwb_synth as S
from parity_util import gpu_cfg_of
from paper_2110_03513_b200 import cwb
ds = S.make("R4", reps=range(6))
pg = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), gpu_cfg_of(ds.cfg))
out = pg.train(torch.as_tensor(ds.Y, device="cuda"), nu=0.05, M=30)
pg.status()
torch.cuda.synchronize()
np.savez(sys.argv[1], **{k: v.cpu().numpy() for k, v in out.items()})
'''
    res = []
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for mode in ("0", "1"):
        path = f"/tmp/h1chunk_{mode}.npz"
        env = dict(os.environ, CWB_H1_CHUNKING=mode, PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]))
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, cwd=root)
        res.append(np.load(path))
    a, b = res
    assert (a["k_trace"] == b["k_trace"]).mean() >= 0.99
    same = (a["k_trace"] == b["k_trace"]).all(0)
    assert np.abs(a["theta_agg"][same] - b["theta_agg"][same]).max() <= 1e-11 * np.abs(a["theta_agg"]).max()


@pytest.mark.parametrize("name,B", [("R2", 128), ("R3", 128), ("R4", 64)])
def test_wide_h1_bitwise_equals_one_column_per_lane(name, B):
    # k_h1w (two replication columns per lane) adds every bin sum in exactly the order of k_h1: the general
    # path's outputs are bitwise the same with CWB_H1_WIDE=0 and 1
    import os
    import subprocess
    import sys
    code = r'''
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
    res = []
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for mode in ("0", "1"):
        path = f"/tmp/h1wide_{name}_{mode}.npz"
        # one sweep in both runs (the row-chunked H1 adds chunk sums: another, equally valid, order)
        env = dict(os.environ, CWB_H1_WIDE=mode, CWB_H1_CHUNKING="0",
                   PYTHONPATH=os.pathsep.join([root, os.path.join(root, "tests")]))
        subprocess.run([sys.executable, "-c", code, path, name, str(B)], check=True, env=env, cwd=root)
        res.append(np.load(path))
    a, b = res
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name,reps", [("R1", range(64)), ("R2", range(0, 1024, 128))])
def test_train_parity_fourth_root_bins(name, reps):
    # n* = ceil(n^(1/4)) (the paper's second bin rule; n* < d leaves Z^T Z rank-deficient)
    import dataclasses
    ds = S.make(name, reps=reps)
    c = dataclasses.replace(ds.cfg, n_star_rule=1)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    assert pg.n_star == O.n_star(c.n, 1)
    out = pg.train(dev(ds.Y), nu=c.nu, M=c.M)
    pg.status()
    g = {k: host(v) for k, v in out.items()}
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    fol = follow_parity(g, po, ds.Y, c.nu, c.M, f"{name} n^(1/4) bins")
    assert fol.sum() <= max(1, 0.01 * c.M * len(reps))
    pg.close()


@pytest.mark.parametrize("ns", [5, 6, 7, 9, 12, 16, 23, 24, 30, 64, 300])
@pytest.mark.parametrize("df", [2.5, 4.0, 5.0])
def test_lambda_calibration_sweep(ns, df):
    # df -> lambda on the definition from rank-deficient (n* < d) to well-determined G
    if df >= ns:
        pytest.skip("df target above the rank")
    rng = np.random.default_rng(ns)
    n = 2000
    X = np.stack([rng.uniform(-1, 2, n), rng.standard_normal(n), rng.exponential(1.0, n)])
    ocfg = O.Config(n_star_rule=2, n_star_fixed=ns, n_knots=20, df=df)
    po = O.Pool(X, ocfg, O.MODE_BINNED)
    pg = cwb.Pool(dev(X), cwb.Config(n_star_rule=2, n_star_fixed=ns, n_knots=20, df=df))
    lam = pg.lam()
    assert np.abs(lam - po.lam).max() <= 1e-9 * np.abs(po.lam).max(), (lam, po.lam)
    pg.close()
