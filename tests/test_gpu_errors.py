"""Error behaviour of the C ABI on bad inputs (include/cwb.h error contracts; round-1 advisor findings):
caller-supplied index vectors out of range, a findBest pool too large for the streaming fit's shared
memory (falls back, same results), learner-sharded contexts on the fused / stream paths, HCWB validation
masks without training or validation rows, and cwb_fit_host's error message."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, TIE_RTOL, close  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def test_bin_mat_vec_rejects_out_of_range_index():
    rng = np.random.default_rng(0)
    ns, n, d = 37, 5000, 24
    Zb = rng.standard_normal((ns, d))
    idx = rng.integers(0, ns, n).astype(np.uint8)
    idx[1234] = ns  # one bin past the end
    R = rng.standard_normal((3, n))
    with pytest.raises(cwb.CwbError) as e:
        cwb.cwb_bin_mat_vec(dev(Zb), dev(idx, torch.uint8), dev(R))
    assert e.value.name == "CWB_EINVAL"
    with pytest.raises(cwb.CwbError) as e:
        cwb.cwb_bin_mat_mat(dev(Zb), dev(idx, torch.uint8))
    assert e.value.name == "CWB_EINVAL"
    # the CUDA context is intact: a valid call afterwards works
    idx[1234] = ns - 1
    out = cwb.cwb_bin_mat_vec(dev(Zb), dev(idx, torch.uint8), dev(R)).cpu().numpy()
    ref = O.bin_mat_vec(Zb, idx.astype(np.int32), R[0])
    ok, err = close(out[0], ref, 1e-12, scale=np.abs(Zb).max() * np.abs(R[0]).sum())
    assert ok, err


def test_find_best_large_n_star_two_columns_falls_back():
    # n* = 4500, B = 2: the streaming fit would need more shared memory than a CTA has; the call must take
    # another findBest path and still match the oracle
    rng = np.random.default_rng(1)
    n = 20000
    X = np.stack([rng.uniform(-3, 5, n), rng.standard_normal(n), rng.exponential(2.0, n)])
    R = np.stack([np.sin(X[0]) + 0.1 * rng.standard_normal(n), X[2] ** 0.5 + rng.standard_normal(n)])
    R -= R.mean(1, keepdims=True)
    pg = cwb.Pool(dev(X), cwb.Config(n_star_rule=2, n_star_fixed=4500))
    po = O.Pool(X, O.Config(n_star_rule=2, n_star_fixed=4500), O.MODE_BINNED)
    k, th, sse = (t.cpu().numpy() for t in pg.find_best(dev(R)))
    pg.status()
    for b in range(2):
        ko, tho, sseo, _, gap = po.find_best(R[b])
        assert k[b] == ko or gap / sseo <= TIE_RTOL
        if k[b] == ko:
            ok, e = close(th[b], tho, RTOL, scale=np.abs(tho).max())
            assert ok, e
    pg.close()


def test_learner_sharded_context_rejects_fused_and_stream_paths():
    rng = np.random.default_rng(2)
    X = rng.uniform(0, 1, (4, 500))
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=4))

    def allreduce(buf, count, stream):  # world 1: the sum over ranks is the buffer itself
        return None
    comm = cwb.Comm(0, 1, fn=allreduce)
    pg.attach_learners(comm)
    for p in (0, 1):
        with pytest.raises(cwb.CwbError) as e:
            pg.set_path(p)
        assert e.value.name == "CWB_EUNSUPPORTED"
    pg.set_path(2)
    pg.close()


@pytest.mark.parametrize("which", ["no_validation", "no_training"])
@pytest.mark.parametrize("path", [1, 2])
def test_hcwb_mask_without_both_sets(which, path):
    rng = np.random.default_rng(3)
    n = 400
    X = rng.uniform(0, 1, (3, n))
    Y = rng.standard_normal((4, n))
    vm = np.zeros(n, np.uint8) if which == "no_validation" else np.ones(n, np.uint8)
    pg = cwb.Pool(dev(X), cwb.Config(n_knots=4))
    pg.set_path(path)
    with pytest.raises(cwb.CwbError) as e:
        pg.train_hcwb(dev(Y), dev(vm, torch.uint8), M=10)
        pg.status()
    assert e.value.name == "CWB_EINVAL"
    pg.close()


def test_fit_host_error_message_survives_the_context():
    rng = np.random.default_rng(4)
    X = rng.uniform(0, 1, (2, 100))
    Y = rng.standard_normal((2, 100))
    Y[1, 7] = np.nan
    with pytest.raises(cwb.CwbError) as e:
        cwb.cwb_fit_host(X, Y, cwb.Config(n_knots=4), nu=0.1, M=5)
    assert e.value.name == "CWB_ENONFINITE"
    assert "ENONFINITE" in str(e.value) and len(str(e.value)) > len("CWB_ENONFINITE: ")
