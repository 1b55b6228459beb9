"""Host-side wall time of the C-ABI calls of one bench step (R1): cwb_init, cwb_train (enqueue),
stream sync, cwb_free, and cwb_fit_host end to end.  usage: python tools/host_overhead.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cwb_synth as S  # noqa: E402
from paper_2110_03513_b200 import cwb  # noqa: E402

c = S.CONFIGS["R1"]
ds = S.make(c)
X = torch.as_tensor(ds.X, device="cuda")
Y = torch.as_tensor(ds.Y, device="cuda")
cfg = cwb.Config(batch_hint=c.B)
torch.cuda.synchronize()
T = {"init": [], "train_enqueue": [], "sync": [], "free": [], "total": []}
for it in range(15):
    t0 = time.perf_counter()
    p = cwb.Pool(X, cfg)
    t1 = time.perf_counter()
    out = p.train(Y, nu=c.nu, M=c.M)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    p.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if it >= 5:
        for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)):
            T[k].append(v * 1e3)
for k, v in T.items():
    print(f"{k:14s} {np.median(v):.3f} ms (median of {len(v)})")
# cwb_fit_host end to end
lib = cwb.load()
Xh = torch.as_tensor(ds.X).pin_memory()
Yh = torch.as_tensor(ds.Y).pin_memory()
K, n, B, M, d = c.K, c.n, c.B, c.M, 24
outs = [torch.empty(s, dtype=dt).pin_memory() for s, dt in (((B,), torch.float64), ((B, K, d), torch.float64),
                                                            ((M, B), torch.int32), ((M, B), torch.float64),
                                                            ((M, B), torch.float64))]
ccfg = cfg.c()
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
ts = []
for it in range(15):
    t0 = time.perf_counter()
    rc = lib.cwb_fit_host(P(Xh), n, K, C.byref(ccfg), P(Yh), B, float(c.nu), M, *[P(o) for o in outs],
                          C.c_void_p(torch.cuda.current_stream().cuda_stream))
    t1 = time.perf_counter()
    assert rc == 0
    if it >= 5:
        ts.append((t1 - t0) * 1e3)
print(f"cwb_fit_host   {np.median(ts):.3f} ms (median, host wall clock incl. sync)")
