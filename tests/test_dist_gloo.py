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
