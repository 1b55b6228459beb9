"""The chunked bin inversion (k_csrc_*, n > 65536) against the one-CTA-per-learner k_csr
(CWB_CSR_CHUNKED=0, run in a subprocess): a stable counting sort is unique, so the pools --
and every training output built on them -- must be bit-identical."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2110_03513_b200 import cwb
n, K, ns, path = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
rng = np.random.default_rng(5)
X = np.stack([rng.uniform(-3, 7, n) if k % 2 == 0 else rng.standard_normal(n) for k in range(K)])
X[1, : n // 4] = X[1, 0]  # a heavy bin
Y = np.stack([np.sin(X[0]) + 0.3 * X[1] + rng.standard_normal(n) for _ in range(3)])
pg = cwb.Pool(torch.as_tensor(X, device="cuda"), cwb.Config(n_star_rule=2, n_star_fixed=ns, n_knots=12))
pg.set_path(path)
out = pg.train(torch.as_tensor(Y, device="cuda"), nu=0.1, M=15)
pg.status()
np.savez(sys.argv[6], **{k: v.cpu().numpy() for k, v in out.items()},
         **{"pool_" + k: v.cpu().numpy() for k, v in pg.pool().items()})
'''


def run(env_extra, args, out):
    env = dict(os.environ, **env_extra)
    subprocess.run([sys.executable, "-c", SCRIPT, ROOT] + [str(a) for a in args] + [out], env=env, check=True,
                   timeout=300)
    return np.load(out)


@pytest.mark.parametrize("n,K,ns,path", [(70001, 3, 265, 2), (200000, 4, 448, 2), (131072, 2, 3000, 2),
                                         (100000, 3, 317, 0)])
def test_chunked_bin_inversion_bit_identical(tmp_path, n, K, ns, path):
    a = run({"CWB_CSR_CHUNKED": "0"}, [n, K, ns, path], str(tmp_path / "a.npz"))
    b = run({}, [n, K, ns, path], str(tmp_path / "b.npz"))
    for k in a.files:
        assert (a[k] == b[k]).all(), k
