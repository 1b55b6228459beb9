"""Per-phase cycle counts of the fused kernel (CTA 0) and event time of cwb_train.
usage: python tools/phase_timing.py [R1 [B [cwb|bernoulli|acwb|hcwb]]]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cwb_synth as S
from paper_2110_03513_b200 import cwb

name = sys.argv[1] if len(sys.argv) > 1 else "R1"
c = S.CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else c.B
ds = S.make(c, reps=range(B))
X = torch.as_tensor(ds.X, device="cuda")
Y = torch.as_tensor(ds.Y, device="cuda")
pool = cwb.Pool(X, cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                              degree=c.degree, df=c.df))
algo = sys.argv[3] if len(sys.argv) > 3 else "cwb"
cyc = torch.zeros(4, dtype=torch.int64, device="cuda")
if algo == "bernoulli":
    Y = torch.as_tensor(S.binary_targets(ds), device="cuda")
    run = lambda: pool.train_bernoulli(Y, nu=c.nu, M=c.M)
elif algo == "acwb":
    run = lambda: pool.train_acwb(Y, nu=c.nu, gamma=0.0034, M=c.M)
elif algo == "hcwb":
    vm = torch.as_tensor(S.validation_mask(c.n), device="cuda")
    run = lambda: pool.train_hcwb(Y, vm, nu=c.nu, gamma=0.037, pat0=5, M=c.M)
else:
    out = pool.train(Y, nu=c.nu, M=c.M)
    run = lambda: pool.train(Y, nu=c.nu, M=c.M, out=out)
run()
pool.set_phase_timing(cyc)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record()
pool.status(); torch.cuda.synchronize()
ph = cyc.cpu().tolist()
print(f"{name} {algo} B={B} train {e0.elapsed_time(e1)*1e3:.1f} us; CTA0 cycles/iter A={ph[0]/c.M:.0f} B={ph[1]/c.M:.0f} "
      f"C={ph[2]/c.M:.0f} D={ph[3]/c.M:.0f} total={sum(ph)/c.M:.0f}")
