"""GPU tests of row sharding (include/cwb.h "row sharding") through the
C ABI: cwb_comm_init / cwb_comm_init_fn + cwb_attach_comm, then cwb_train / cwb_find_best on the local
row block.

* world 1 over a real NCCL communicator: the same bytes as the unsharded general path (the
  all-reduce of one rank is the identity and every other step is the same kernel).
* world 2 and 3 on the one GPU: one context per rank, each driven by its own host thread;
  the collective is a host-side rendezvous that sums the ranks' device buffers in rank
  order (cwb_comm_init_fn).  No kernel waits on another rank's kernel (the ranks
  only meet on the host), so this is the multi-rank data path without multi-GPU
  hardware.  Checked against the oracle on the FULL data with the parity rules of
  tests/parity_util.py (sums in another order: within tolerance, not bitwise).
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, assert_train_parity, cfg_of, close, gpu_cfg_of  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402
from paper_2110_03513_b200 import dist as D  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


class ThreadAllReduce:
    """Sum over W host threads (one per emulated rank) of a device fp64 buffer, rank order."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world, timeout=120)
        self.parts = [None] * world
        self.calls = [0] * world

    def fn(self, rank):
        def f(ptr, count, stream):
            torch.cuda.synchronize()
            t = D.device_view(ptr, count, DEV)
            self.parts[rank] = t.clone()
            self.bar.wait()
            tot = self.parts[0].clone()
            for r in range(1, self.world):
                tot += self.parts[r]
            self.bar.wait()  # every rank has read the parts before the next round writes them
            t.copy_(tot)
            torch.cuda.synchronize()
            self.calls[rank] += 1
        return f


def run_ranks(world, body):
    """body(rank) in one thread per rank; re-raises the first failure."""
    res, errs = [None] * world, []

    def run(r):
        try:
            res[r] = body(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    if errs:
        raise errs[0]
    assert all(not t.is_alive() for t in th), "a rank hung"
    return res


def gpu_train(p, Y, nu, M):
    out = p.train(dev(Y), nu=nu, M=M)
    p.status()
    return {k: host(v) for k, v in out.items()}


@pytest.mark.parametrize("name", ["R0", "R1"])
def test_rows_world1_nccl_equals_unsharded(name):
    ds = S.make(name, reps=np.arange(min(S.CONFIGS[name].B, 64)))
    c = ds.cfg
    ref = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    ref.set_path(2)
    g0 = gpu_train(ref, ds.Y, c.nu, c.M)
    p = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    comm = cwb.Comm(0, 1, unique_id=cwb.cwb_comm_unique_id())
    p.attach(comm)
    assert p.rows() == (0, ds.X.shape[1], 0, 1)
    g1 = gpu_train(p, ds.Y, c.nu, c.M)
    for k in g0:
        assert np.array_equal(g0[k], g1[k]), f"{name}: {k} differs"
    # find_best (B > 4: the general, not the narrow, unsharded path)
    R = dev(ds.Y[:8] - ds.Y[:8].mean(axis=1, keepdims=True))
    a = [host(t) for t in ref.find_best(R)]
    b = [host(t) for t in p.find_best(R)]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # the communicator serves a second context
    p2 = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    p2.attach(comm)
    g2 = gpu_train(p2, ds.Y, c.nu, c.M)
    assert np.array_equal(g0["theta_agg"], g2["theta_agg"])


@pytest.mark.parametrize("name,world", [("R0", 2), ("R1", 2), ("R1", 3)])
def test_rows_multi_rank_parity(name, world):
    reps = np.arange(min(S.CONFIGS[name].B, 32))
    ds = S.make(name, reps=reps)
    c = ds.cfg
    n = ds.X.shape[1]
    o = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED).train(ds.Y, nu=c.nu, M=c.M, threads=8)
    ar = ThreadAllReduce(world)
    pools = [cwb.Pool(dev(ds.X), gpu_cfg_of(c)) for _ in range(world)]
    comms = [cwb.Comm(r, world, fn=ar.fn(r)) for r in range(world)]
    for r, p in enumerate(pools):
        p.attach(comms[r])
        blk = D.row_block(n, r, world)
        assert p.rows() == (blk.start, len(blk), r, world)

    def body(r):
        blk = D.row_block(n, r, world)
        return gpu_train(pools[r], ds.Y[:, blk.start:blk.stop], c.nu, c.M)

    res = run_ranks(world, body)
    assert ar.calls == [c.M + 2] * world  # offsets, one per iteration, the last risk
    for r in range(1, world):  # every rank holds the same model
        for k in ("k_trace", "theta_agg", "offset", "sse_trace", "risk_trace"):
            assert np.array_equal(res[0][k], res[r][k]), f"rank {r}: {k}"
    assert_train_parity(res[0], o, n, f"{name} rows x{world}")


def test_rows_find_best_parity():
    ds = S.make("R1", reps=np.arange(6))
    c = ds.cfg
    n = ds.X.shape[1]
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    R = ds.Y - ds.Y.mean(axis=1, keepdims=True)
    world = 2
    ar = ThreadAllReduce(world)
    pools = [cwb.Pool(dev(ds.X), gpu_cfg_of(c)) for _ in range(world)]
    comms = [cwb.Comm(r, world, fn=ar.fn(r)) for r in range(world)]
    for r, p in enumerate(pools):
        p.attach(comms[r])

    def body(r):
        blk = D.row_block(n, r, world)
        k, th, sse = pools[r].find_best(dev(R[:, blk.start:blk.stop]))
        return host(k), host(th), host(sse)

    res = run_ranks(world, body)
    for b in range(R.shape[0]):
        ko, tho, sseo, _, _ = po.find_best(R[b])
        assert res[0][0][b] == ko
        ok, e = close(res[0][1][b], tho, RTOL)
        assert ok, e
        ok, e = close(res[0][2][b], sseo, RTOL)
        assert ok, e


def test_rows_errors():
    ds = S.make("R0", reps=np.arange(2))
    c = ds.cfg
    with pytest.raises(cwb.CwbError) as e:
        cwb.Comm(2, 2, fn=lambda *a: None)
    assert e.value.name == "CWB_EINVAL"
    p2 = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    big = ds.X.shape[1] + 1
    with pytest.raises(cwb.CwbError) as e:
        p2.attach(cwb.Comm(0, big, fn=lambda *a: None))
    assert e.value.name == "CWB_EINVAL"
    comm = cwb.Comm(0, 1, unique_id=cwb.cwb_comm_unique_id())
    p3 = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    p3.attach(comm)
    with pytest.raises(cwb.CwbError) as e:
        p3.attach(comm)
    assert e.value.name == "CWB_EINVAL"  # (errors are sticky: p3 now reports it on every call)
    p5 = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    p5.attach(comm)
    with pytest.raises(cwb.CwbError) as e:
        p5.train_acwb(dev(ds.Y), M=3)
    assert e.value.name == "CWB_EUNSUPPORTED"
    # a failing collective surfaces as CWB_ENCCL
    p4 = cwb.Pool(dev(ds.X), gpu_cfg_of(c))

    def bad(ptr, count, stream):
        raise RuntimeError("collective down")
    p4.attach(cwb.Comm(0, 1, fn=bad))
    with pytest.raises(cwb.CwbError) as e:
        p4.train(dev(ds.Y), M=2)
    assert e.value.name == "CWB_ENCCL"
