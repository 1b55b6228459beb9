import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2110_03513_b200.cwb as cwb
cwb.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpurun_dbg_libcwb.so")
import cwb_synth as S
for name in ["R1", "R0"]:
    ds = S.make(name, reps=[0]); c = ds.cfg
    p = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots))
    p.status(); torch.cuda.synchronize()
    print(name, p.lam())
