"""GPU tests of learner sharding (cwb_attach_comm_learners, SURVEY 8(e) alternative): every rank
holds all rows and learners and fits its block of learners; one all-reduce per iteration gathers
the candidates.  The results are bitwise those of the unsharded per-iteration kernels (same
arithmetic per learner, same argmin with the lowest k on ties).  world 2 / 3 run as host threads
on the one GPU with the host-side rendezvous collective of tests/test_gpu_rows.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from parity_util import gpu_cfg_of  # noqa: E402
from test_gpu_rows import ThreadAllReduce, dev, gpu_train, host, run_ranks  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402


@pytest.mark.parametrize("name,world", [("R0", 1), ("R0", 2), ("R1", 2), ("R1", 3), ("R2", 3)])
def test_learner_sharding_equals_unsharded(name, world):
    reps = np.arange(min(S.CONFIGS[name].B, 40))
    ds = S.make(name, reps=reps)
    c = ds.cfg
    M = min(c.M, 80)
    ref = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    ref.set_path(2)
    g0 = gpu_train(ref, ds.Y, c.nu, M)
    if world == 1:
        comms = [cwb.Comm(0, 1, unique_id=cwb.cwb_comm_unique_id())]
        ar = None
    else:
        ar = ThreadAllReduce(world)
        comms = [cwb.Comm(r, world, fn=ar.fn(r)) for r in range(world)]
    pools = [cwb.Pool(dev(ds.X), gpu_cfg_of(c)) for _ in range(world)]
    for r, p in enumerate(pools):
        p.attach_learners(comms[r])
    res = run_ranks(world, lambda r: gpu_train(pools[r], ds.Y, c.nu, M))
    if ar is not None:
        assert ar.calls == [M] * world  # one all-reduce per iteration
    for r in range(world):
        for k in g0:
            assert np.array_equal(g0[k], res[r][k]), f"rank {r}: {k} differs"


def test_learner_sharding_find_best_and_errors():
    ds = S.make("R1", reps=np.arange(6))
    c = ds.cfg
    R = dev(ds.Y - ds.Y.mean(axis=1, keepdims=True))
    ref = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    ref.set_path(2)
    a = [host(t) for t in ref.find_best(R)]
    world = 2
    ar = ThreadAllReduce(world)
    comms = [cwb.Comm(r, world, fn=ar.fn(r)) for r in range(world)]
    pools = [cwb.Pool(dev(ds.X), gpu_cfg_of(c)) for _ in range(world)]
    for r, p in enumerate(pools):
        p.attach_learners(comms[r])
    res = run_ranks(world, lambda r: [host(t) for t in pools[r].find_best(R)])
    for r in range(world):
        for x, y in zip(a, res[r]):
            assert np.array_equal(x, y)
    with pytest.raises(cwb.CwbError) as e:
        pools[0].train_acwb(dev(ds.Y), M=2)
    assert e.value.name == "CWB_EUNSUPPORTED"
    with pytest.raises(cwb.CwbError) as e:
        cwb.Pool(dev(ds.X), gpu_cfg_of(c)).attach_learners(cwb.Comm(0, 11, fn=lambda *a: None))  # world > K
    assert e.value.name == "CWB_EINVAL"
