"""GPU parity of CWB with per-replication cross-validation folds (cwb_train_folds, SURVEY NEXT-4:
0/1 observation weights in binMatMat / binMatVec) against the oracle's
orc_train_folds on seeded folds (cwb_synth.cv_folds)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from parity_util import RTOL, assert_train_parity, cfg_of, close, gpu_cfg_of  # noqa: E402

from paper_2110_03513_b200 import cwb  # noqa: E402

DEV = "cuda:0"


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


@pytest.mark.parametrize("name,reps,M,F", [("R0", None, None, 3), ("R1", None, None, 5), ("R2", range(0, 1024, 101), 60, 5)])
def test_folds_match_oracle(name, reps, M, F):
    ds = S.make(name, reps=reps)
    c = ds.cfg
    M = M or c.M
    B = ds.Y.shape[0]
    fold = S.cv_folds(c.n, F)
    frep = (np.arange(B) % (F + 1) - 1).astype(np.int32)  # -1 (no hold-out), 0 .. F-1
    po = O.Pool(ds.X, cfg_of(c), O.MODE_BINNED)
    o, ov = po.train_folds(ds.Y, fold, F, frep, nu=c.nu, M=M, threads=8)
    pg = cwb.Pool(dev(ds.X), gpu_cfg_of(c))
    out = pg.train_folds(dev(ds.Y), dev(fold, torch.uint8), F, dev(frep, torch.int32), nu=c.nu, M=M)
    pg.status()
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    first, _ = assert_train_parity(g, o, c.n, tag=f"{name} folds")
    for b in range(B):
        m = first[b]
        ok, e = close(g["val_risk_trace"][:m, b], ov[:m, b], RTOL, scale=max(np.abs(ov[:, b]).max(), 1e-300))
        assert ok, f"val risk replication {b}: {e}"
    pg.close()


def test_folds_errors():
    ds = S.make("R1", reps=range(3))
    fold = S.cv_folds(ds.cfg.n, 4)
    for frep, F in ((np.array([0, 4, 1], np.int32), 4), (np.array([0, 0, 0], np.int32), 1)):
        pg = cwb.Pool(dev(ds.X), gpu_cfg_of(ds.cfg))
        fr = fold if F > 1 else np.zeros_like(fold)
        with pytest.raises(cwb.CwbError) as e:
            pg.train_folds(dev(ds.Y), dev(fr, torch.uint8), F, dev(frep, torch.int32), M=2)
            pg.status()
        assert e.value.name == "CWB_EINVAL"
        pg.close()
