"""Per-warp phase timing of the fused kernel at R1 (CTA 0): the spread of the warps' phase-A end times, which warp
ends A last, B after the last A warp, and learner 0's B sub-phases (s-loop, theta, c + delta).  Needs the debug
build of the same sources with -DCWB_PHASE_DEBUG:
    python -c "import os,sys; sys.path.insert(0,'.'); from paper_2110_03513_b200 import build as b; \
      b._build(os.path.join(b.HERE,'libcwb_dbg.so'), os.path.join(b.HERE,'build','dbg'), ['-DCWB_PHASE_DEBUG'], True, False)"
    CWB_LIB=$PWD/paper_2110_03513_b200/libcwb_dbg.so python tools/phase_warps.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import cwb_synth as S
from paper_2110_03513_b200 import cwb
c = S.CONFIGS["R1"]
ds = S.make(c)
pool = cwb.Pool(torch.as_tensor(ds.X, device="cuda"), cwb.Config(batch_hint=c.B))
Y = torch.as_tensor(ds.Y, device="cuda")
out = pool.train(Y, nu=c.nu, M=c.M)
cyc = torch.zeros(80, dtype=torch.int64, device="cuda")
pool.set_phase_timing(cyc)
pool.train(Y, nu=c.nu, M=c.M, out=out)
pool.status(); torch.cuda.synchronize()
v = cyc.cpu().tolist(); M = c.M
print(f"A={v[0]/M:.0f} B={v[1]/M:.0f} C={v[2]/M:.0f} D={v[3]/M:.0f}; A spread over warps {v[4]/M:.0f}; B after the last A warp {v[5]/M:.0f}")
print("last-in-A counts per warp:", v[8:24])
print("mean A end relative to the first warp:", [round(x / M) for x in v[40:56]])
print(f"warp 0 (learner 0) B sub-phases: s-loop {v[60]/M:.0f}, theta {v[61]/M:.0f}, c + delta {v[62]/M:.0f}")
