"""Time cwb_find_best (one findBestBaselearner) on B residual vectors for a config.
The calls are captured in a CUDA graph (no host launch overhead in the measurement).
usage: python tools/findbest_timing.py R3 [B] [reps] [narrow_mode] [flush]
flush=1: no graph; a 256 MiB buffer is written before every call (L2 flushed: the index vectors are
read from HBM, as at sizes above the 126 MB L2) and each call is timed alone with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cwb_synth as S
from paper_2110_03513_b200 import cwb

name = sys.argv[1] if len(sys.argv) > 1 else "R3"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
c = S.CONFIGS[name]
ds = S.make(c, reps=range(B))
X = torch.as_tensor(ds.X, device="cuda")
R = torch.as_tensor(ds.Y - ds.Y.mean(1, keepdims=True), device="cuda")
pool = cwb.Pool(X, cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots))
pool.set_narrow(mode)
flush = len(sys.argv) > 5 and sys.argv[5] == "1"
if flush:
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        pool.find_best(R)
    ts = []
    for i in range(reps):
        buf.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        k, th, sse = pool.find_best(R)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = sorted(ts)[len(ts) // 2]
    K, n = c.K, c.n
    alg = K * n * (1 if pool.n_star <= 256 else 2) + n * B * 8
    print(f"{name} B={B} mode={mode} flushed find_best {us:.1f} us (median of {reps}); alg bytes {alg/1e6:.1f} MB "
          f"-> {alg/us/1e3:.0f} GB/s")
    sys.exit(0)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        k, th, sse = pool.find_best(R)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            k, th, sse = pool.find_best(R)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
K, n = c.K, c.n
idx_bytes = 1 if pool.n_star <= 256 else 2
alg = K * n * idx_bytes + n * B * 8  # index vector + residuals, read once
print(f"{name} B={B} mode={mode} find_best {us:.1f} us; K*n*B={K*n*B:.3g} evals -> {K*n*B/us/1e3:.3g} G evals/s; "
      f"alg bytes {alg/1e6:.1f} MB -> {alg/us/1e3:.0f} GB/s")
