"""Oracle timing variants of SURVEY 8(d) on the host cores: (i) dense mode single thread, (ii) dense
mode all cores, (iii) binned mode (the paper's Algorithm binMatVec) single thread and all cores, in
learner-row evaluations/s on a bounded sample of a workload.  Test infrastructure: times oracle/ as it
stands.  usage: python tools/oracle_timing.py [R1] [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cwb_synth as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "R1"
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
c = S.CONFIGS[name]
cores = os.cpu_count() or 1
oc = O.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots, degree=c.degree, df=c.df)
print(f"# {name}: n={c.n} K={c.K} B={c.B} M={c.M}; host cores {cores}; "
      f"cpu {os.popen('lscpu | grep \"Model name\"').read().strip()}")
for mode, mname in ((O.MODE_DENSE, "dense"), (O.MODE_BINNED, "binned")):
    for th in (1, cores):
        ds1 = S.make(c, reps=range(1))
        pool = O.Pool(ds1.X, oc, mode)
        t0 = time.perf_counter()
        pool.train(ds1.Y, nu=c.nu, M=5, threads=1)
        per = (time.perf_counter() - t0) / 5
        reps = max(1, min(c.B, int(budget * th / max(per * c.M, 1e-9))))
        M = c.M if reps > 1 or per * c.M <= budget else max(1, int(budget / per))
        ds = S.make(c, reps=range(reps))
        t0 = time.perf_counter()
        pool = O.Pool(ds.X, oc, mode)
        pool.train(ds.Y, nu=c.nu, M=M, threads=th)
        dt = time.perf_counter() - t0
        ev = c.K * c.n * reps * M
        print(f"{mname:6s} threads {th:3d}: {ev / dt:.3e} evals/s  ({reps} replications x M={M}, {dt:.2f} s, "
              f"pool build included)")
