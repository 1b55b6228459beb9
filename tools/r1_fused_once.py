"""Two cwb_train calls at R1 (B = 256) on the fused kernel, for ncu captures of k_train_fused."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

ds = S.make("R1")
c = ds.cfg
pool = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), cwb.Config(batch_hint=c.B))
Y = torch.as_tensor(ds.Y, device="cuda")
for _ in range(2):
    pool.train(Y, nu=c.nu, M=c.M)
pool.status()
torch.cuda.synchronize()
print("ok")
