"""world_size-2 tests of the multi-process host logic on CPU (gloo): replication sharding,
max-over-ranks timing and result gathering.  The compute is the CPU oracle (test
infrastructure); what is under test is that sharding replications over ranks and
gathering the per-rank results reproduces the single-process run bit for bit, which is
what the GPU path relies on (no collective on the data path)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from paper_2110_03513_b200 import dist as D  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size),
                      LOCAL_RANK=str(rank))
    try:
        import cwb_synth as S
        from oracle import oracle as O
        w = D.world_from_env()
        D.init_process_group(w, "gloo")
        cfg = S.CONFIGS["R0"]
        reps = D.replication_block(4, w.rank)              # weak scaling: 4 replications per rank
        ds = S.make(cfg, reps=reps)
        pool = O.Pool(ds.X, O.Config(n_star_rule=cfg.n_star_rule, n_star_fixed=cfg.n_star_fixed,
                                     n_knots=cfg.n_knots), O.MODE_BINNED)
        res = pool.train(ds.Y, nu=cfg.nu, M=cfg.M)
        kt = D.gather_rows(torch.as_tensor(np.ascontiguousarray(res.k_trace.T)), w)      # [B_total, M]
        agg = D.gather_rows(torch.as_tensor(res.theta_agg), w)                          # [B_total, K, d]
        # the packed one-collective gather bench.py runs at the end of every sharded step
        full = D.gather_results({"offset": torch.as_tensor(res.offset), "theta_agg": torch.as_tensor(res.theta_agg),
                                 "k_trace": torch.as_tensor(res.k_trace), "sse_trace": torch.as_tensor(res.sse_trace),
                                 "risk_trace": torch.as_tensor(res.risk_trace)}, w)
        assert (full["theta_agg"].numpy() == agg.numpy()).all()
        assert (full["k_trace"].numpy().T == kt.numpy()).all() and full["k_trace"].dtype == torch.int32
        assert full["sse_trace"].shape == (cfg.M, 4 * size) and full["offset"].shape == (4 * size,)
        tmax = D.max_over_ranks(float(10 + w.rank), w)
        D.barrier(w)
        strong = [list(D.split_replications(7, size, r)) for r in range(size)]
        if w.rank == 0:
            q.put(("ok", kt.numpy(), agg.numpy(), tmax, strong))
        import torch.distributed as dist
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put(("err", repr(e)))


def test_replication_sharding_matches_single_process():
    size = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert out[0] == "ok", out
    _, kt, agg, tmax, strong = out
    import cwb_synth as S
    from oracle import oracle as O
    cfg = S.CONFIGS["R0"]
    ds = S.make(cfg, reps=range(8))
    pool = O.Pool(ds.X, O.Config(n_star_rule=cfg.n_star_rule, n_star_fixed=cfg.n_star_fixed, n_knots=cfg.n_knots),
                  O.MODE_BINNED)
    ref = pool.train(ds.Y, nu=cfg.nu, M=cfg.M)
    assert (kt == ref.k_trace.T).all()
    assert (agg == ref.theta_agg).all()        # bitwise: replications are independent
    assert tmax == 11.0                         # max over ranks
    assert strong == [[0, 1, 2, 3], [4, 5, 6]]


def test_split_and_block_host_logic():
    for total in range(0, 40):
        for size in range(1, 9):
            seen = [b for r in range(size) for b in D.split_replications(total, size, r)]
            assert seen == list(range(total))
    assert list(D.replication_block(3, 2)) == [6, 7, 8]
    with pytest.raises(ValueError):
        D.split_replications(4, 2, 2)
    w = D.World()
    assert D.max_over_ranks(3.5, w) == 3.5


# ----------------------------------------------------------------- row sharding
# The decomposition the GPU row-sharded path (include/cwb.h "row sharding") relies on,
# run with the oracle's binMatVec / Cholesky solve as its steps over a world-2 gloo
# group: every rank holds the full pool and a row block; per iteration the per-rank
# s = Zb^T u (binMatVec is a sum over rows) and r^T r are all-reduced, the
# selection runs redundantly, the update touches local rows.  It must reproduce the
# single-process oracle run.

def _rows_worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size),
                      LOCAL_RANK=str(rank))
    try:
        import torch.distributed as dist
        import cwb_synth as S
        from oracle import oracle as O
        w = D.world_from_env()
        D.init_process_group(w, "gloo")
        uid = D.broadcast_bytes(bytes(range(128)) if w.rank == 0 else None, w)
        cfg = S.CONFIGS["R0"]
        ds = S.make(cfg, reps=range(3))
        pool = O.Pool(ds.X, O.Config(n_star_rule=cfg.n_star_rule, n_star_fixed=cfg.n_star_fixed,
                                     n_knots=cfg.n_knots), O.MODE_BINNED)
        K, n, d, B, M, nu = pool.K, pool.n, pool.d, ds.Y.shape[0], cfg.M, cfg.nu
        blk = D.row_block(n, w.rank, w.size)
        idx = pool.idx[:, blk.start:blk.stop]
        Y = ds.Y[:, blk.start:blk.stop]
        t = torch.as_tensor(Y.sum(axis=1))
        dist.all_reduce(t)
        f0 = t.numpy() / n
        R = Y - f0[:, None]
        rr_loc = (R * R).sum(axis=1)
        A = [pool.G[k] + pool.lam[k] * pool.D for k in range(K)]
        ks = np.zeros((M, B), dtype=np.int64)
        agg = np.zeros((B, K, d))
        for m in range(M):
            s_loc = np.array([[O.bin_mat_vec(pool.Zb[k], idx[k], R[b]) for k in range(K)] for b in range(B)])
            pack = torch.as_tensor(np.concatenate([s_loc.ravel(), rr_loc]))
            dist.all_reduce(pack)
            s = pack[: B * K * d].numpy().reshape(B, K, d)
            rr = pack[B * K * d:].numpy()
            for b in range(B):
                th = [O.chol_solve(A[k], s[b, k]) for k in range(K)]
                sse = [rr[b] - 2 * th[k] @ s[b, k] + th[k] @ pool.G[k] @ th[k] for k in range(K)]
                k = int(np.argmin(sse))
                ks[m, b] = k
                agg[b, k] += nu * th[k]
                R[b] -= nu * (pool.Zb[k][idx[k]] @ th[k])
            rr_loc = (R * R).sum(axis=1)
        if w.rank == 0:
            q.put(("ok", ks, agg, f0, uid))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put(("err", traceback.format_exc()))


def test_row_sharding_decomposition_matches_single_process():
    size = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert out[0] == "ok", out
    _, ks, agg, f0, uid = out
    import cwb_synth as S
    from oracle import oracle as O
    cfg = S.CONFIGS["R0"]
    ds = S.make(cfg, reps=range(3))
    pool = O.Pool(ds.X, O.Config(n_star_rule=cfg.n_star_rule, n_star_fixed=cfg.n_star_fixed, n_knots=cfg.n_knots),
                  O.MODE_BINNED)
    ref = pool.train(ds.Y, nu=cfg.nu, M=cfg.M)
    assert uid == bytes(range(128))
    assert (ks == ref.k_trace).all()
    np.testing.assert_allclose(f0, ref.offset, rtol=1e-13)
    np.testing.assert_allclose(agg, ref.theta_agg, rtol=1e-9, atol=1e-12 * np.abs(ref.theta_agg).max())


def test_row_block_partition():
    for n in range(1, 60):
        for world in range(1, min(n, 9) + 1):
            rows = [i for r in range(world) for i in D.row_block(n, r, world)]
            assert rows == list(range(n))
            sizes = [len(D.row_block(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.row_block(3, 0, 4)
    assert D.broadcast_bytes(b"abc", D.World()) == b"abc"
