#!/usr/bin/env python
"""Benchmark of the B200 binned-CWB engine (arXiv 2110.03513).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config R3] [--impl ours|reference]

One STEP = the whole hot path on one batch: cwb_init (binning, bin inversion,
basis, G, df->lambda, cached inverse) + cwb_train (M boosting iterations for
the B replications of the workload), inputs resident in HBM.  Metric (the
reshaped BASELINE.json metric): learner-row evaluations per
second = K*n*B*M / step time (one evaluation = one (learner, row,
replication) contribution of the binMatVec scatter of P:L899-901).

Timing: W warm-up steps, then K steps, each bracketed by CUDA events on the
launching stream; L2 is flushed (256 MiB write) between steps outside the
events; barrier + synchronize around the timed region; max over ranks.
N > 1 (torchrun): replications are sharded (weak scaling, every rank its own
B replications, no collective on the data path); with --shard rows the rows
are (strong scaling: the B replications of the workload on n rows split over
the ranks, one NCCL all-reduce of (K d + 1) x B doubles per iteration issued
by libcwb).

Default workload: R3 (n = 200,000, K = 66, B = 512, M = 200), the largest rung
of the ladder that runs on one GPU (P:L1047 scale); R1 and
the others by --config.

Roofline: for the dominant kernel of the step (k_train_fused
when the whole run is one persistent launch, else the binMatVec phase H1 of the
per-iteration path, timed with CUDA events that libcwb records around it),
roofline time = max(bytes_alg / HBM, adds_alg / DADD) with bytes_alg =
K n ceil(log2 n* / 8) + n B 8 (H1 reads the index vectors and the residuals;
+ n B 8 for the residual write of a whole iteration) and adds_alg = K n B;
frac = roofline time / kernel time.  HBM = MEASURED_PEAKS.json's copy bandwidth,
DADD = the measured issue rate in profiles/peaks_fp64.json (tools/peaks.py).

--impl reference times the CPU oracle (oracle/, plain fp64 C) on a bounded
sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import cwb_synth as S  # noqa: E402

METRIC = "learner-row evaluations/s (K*n*B per boosting iteration) and boosting iterations/s"
UNIT = "evals/s"


def alg_ops_per_rep_iter(c, n_star, d, unbinned=False):
    """Algorithmic fp64 add/FMA operations per replication-iteration of the fused kernel."""
    K, n = c.K, c.n
    if unbinned:  # 4-tap scatter per (learner, row), fit/SSE as binned, r -= nu Z theta with 4 taps
        return 4 * K * n + K * d * d + 5 * K * d + 4 * n + 2 * n + d
    h1 = K * n                      # binMatVec sums: one add per (learner, row)
    h2 = 4 * K * n_star             # s = Zb^T u, 4 non-zeros per design point
    h3 = K * d * d                  # theta = A^-1 s
    h4 = 5 * K * d                  # c = C^T theta (4 per coefficient), |c|^2
    h6 = 4 * n_star + 2 * n + d     # zhat, r update + r^T r, theta_agg
    return h1 + h2 + h3 + h4 + h6


# measured conflict-free shared-memory gather ceiling (profiles/ubench_smem_gather.txt):
# 16-byte lane-loads (RB = 2 replications per row) and 8-byte lane-loads (RB = 1) per clock per SM
GATHER_LANE_LOADS_PER_CLK = {2: 7.1, 1: 12.7}


def load_peaks():
    """MEASURED_PEAKS.json (driver-written: HBM copy GB/s, clocks) + profiles/peaks_fp64.json
    (tools/peaks.py on this pool's B200: DADD / DFMA issue rate, L2 / HBM read, DGEMM)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        peaks, src = json.load(open(p)), "measured"
    except Exception:
        peaks, src = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"
    try:
        f = json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64.json")))
        m = {r["what"]: r for r in f["measurements"]}
        peaks["dadd_tops"] = m["dadd"]["ops_per_s"] / 1e12
        peaks["dfma_tops"] = m["dfma"]["ops_per_s"] / 1e12
        peaks["l2_read_gbs"] = max([m["l2_read"]["gb_per_s"]] + [r["gb_per_s"] for k, r in m.items()
                                                                 if k.startswith("l2_read8_")])
        peaks["hbm_read_gbs"] = m["hbm_read"]["gb_per_s"]
        peaks["dgemm_tflops"] = m["dgemm_cublas"]["tflops"]
        peaks["fp64_src"] = "measured (profiles/peaks_fp64.json)"
    except Exception:  # datasheet product, said so in the line
        peaks["dadd_tops"] = 148 * 64 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e-6
        peaks["fp64_src"] = "datasheet (148 SM x 64 lanes x clock): profiles/peaks_fp64.json missing"
    return peaks, src


def idx_bytes_of(n_star):
    return 1 if n_star <= 256 else 2   # ceil(log2 n* / 8)


def sec8d_roofline(K, n, B, n_star, peaks, kernel_s, units, what, bytes_extra=0):
    """roofline time = max(bytes_alg / HBM, adds_alg / DADD) of `units` launches-worth of
    work (H1 of one iteration: K n idx bytes + n B 8 residual bytes, K n B adds); frac = that / kernel time."""
    bytes_alg = units * (K * n * idx_bytes_of(n_star) + n * B * 8 + bytes_extra)
    adds_alg = units * K * n * B
    hbm = float(peaks["hbm_gbs"]) * 1e9
    dadd = float(peaks["dadd_tops"]) * 1e12
    t_hbm, t_dadd = bytes_alg / hbm, adds_alg / dadd
    bound = "hbm" if t_hbm >= t_dadd else "alu"
    if bound == "hbm":
        achieved, peak, unit = bytes_alg / kernel_s / 1e9, hbm / 1e9, "GB/s"
    else:
        achieved, peak, unit = adds_alg / kernel_s / 1e12, dadd / 1e12, "TFLOP/s"  # one fp64 add = one flop
    return {"bound": bound, "kernel": what, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": max(t_hbm, t_dadd) / kernel_s,
            "terms": {"bytes_alg": bytes_alg, "adds_alg": adds_alg, "t_hbm_ms": t_hbm * 1e3,
                      "t_dadd_ms": t_dadd * 1e3, "t_kernel_ms": kernel_s * 1e3,
                      "hbm_gbs": hbm / 1e9, "dadd_tops": dadd / 1e12}}


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _names(self, mask):
        N = self.N
        table = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
                 "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                 "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}
        return {k for k, v in table.items() if mask & v}

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                self.reasons |= self._names(N.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def dist_env():
    from paper_2110_03513_b200 import dist as D
    w = D.world_from_env()
    return w.size, w.rank, w.local_rank


_ORACLE_PLAN = {}


def oracle_sample(cfg, seconds_target=12.0, threads=None, algo="cwb", unbinned=False):
    """Time the oracle as it stands (binned mode = the paper's Algorithm binMatVec; unbinned mode for
    --unbinned) on a bounded sample of the workload, running the same algorithm as the GPU arm."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    c = cfg
    oc = O.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                  degree=c.degree, df=c.df)
    mode = O.MODE_UNBINNED if unbinned else O.MODE_BINNED
    fits = 2 if algo in ("acwb", "hcwb") else 1  # evaluations per iteration as in the GPU arm (HCWB: upper bound)

    def run(pool, ds, M, th):
        Y = S.binary_targets(ds) if algo == "bernoulli" else ds.Y
        if algo == "acwb":
            return pool.train_acwb(Y, nu=c.nu, gamma=0.0034, M=M, threads=th)
        if algo == "hcwb":
            return pool.train_hcwb(Y, S.validation_mask(c.n), nu=c.nu, gamma=0.037, pat0=5, M=M, threads=th)
        if algo == "bernoulli":
            return pool.train_bernoulli(Y, nu=c.nu, M=M, threads=th)
        return pool.train(Y, nu=c.nu, M=M, threads=th)

    # probe (first call only): one replication, a few iterations, on a pool built once; sizes the sample so that
    # its training part takes about seconds_target on `threads` cores (at least one replication per core
    # is free: the replications run in parallel)
    key = (c.name, algo, unbinned, threads, seconds_target)
    if key not in _ORACLE_PLAN:
        ds1 = S.make(c, reps=range(1))
        t0 = time.perf_counter()
        pool = O.Pool(ds1.X, oc, mode)
        t_init = time.perf_counter() - t0
        M_probe = max(1, min(c.M, 5))
        t0 = time.perf_counter()
        run(pool, ds1, M_probe, 1)
        per_rep_iter = (time.perf_counter() - t0) / M_probe
        del pool
        reps = int(max(1, seconds_target * threads / max(per_rep_iter * c.M, 1e-9)))
        reps = max(min(reps, c.B), min(threads, c.B), 1)
        _ORACLE_PLAN[key] = (reps, S.make(c, reps=range(reps)))
    reps, ds = _ORACLE_PLAN[key]
    # one step: pool build (the GPU arm's cwb_init) + M iterations of the sampled replications
    t0 = time.perf_counter()
    pool = O.Pool(ds.X, oc, mode)
    t_init = time.perf_counter() - t0
    run(pool, ds, c.M, threads)
    dt = time.perf_counter() - t0
    evals = fits * c.K * c.n * reps * c.M
    kind = "unbinned mode" if unbinned else "binned mode (Algorithm binMatVec, P:L898-904)"
    return {"value": evals / dt, "unit": UNIT, "cores": min(threads, reps), "kind": "oracle",
            "sample": f"{c.name}: {reps} of {c.B} replications x M={c.M} iterations, oracle {algo}, {kind}, "
                      f"pool build included ({t_init:.2f} s); {dt:.2f} s",
            "seconds": dt, "init_s": t_init}


def run_reference(args, cfg):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    res = []
    for i in range(args.warmup + args.steps):
        r = oracle_sample(cfg, seconds_target=args.ref_seconds, threads=threads, algo=args.algo,
                          unbinned=args.unbinned)
        if i >= args.warmup:
            res.append(r)
    v = float(np.mean([r["value"] for r in res]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean([r["seconds"] for r in res]) * 1e3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (paper Sec. 4.1.1 generator, seeded)",
            "config": dict(workload_config(cfg, O.n_star(cfg.n, cfg.n_star_rule, cfg.n_star_fixed),
                                           cfg.n_knots + cfg.degree + 1), algo=args.algo, shard="replications",
                           learners="unbinned" if args.unbinned else "binned", parallelism=f"replications{args.gpus}"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": res[0]["cores"], "kind": "oracle",
                             "sample": res[0]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def r1_rung(devname, peaks, steps=20, warmup=5):
    """The R1 rung (n = 1,331, K = 10, B = 256, M = 200: the latency-bound rung, one persistent k_train_fused
    launch per cwb_train) measured like the headline step (fresh pool per step, L2 flushed between steps, CUDA
    events), with the SURVEY 8(d) roofline of its kernel -- an extra key of the default line."""
    import torch
    from paper_2110_03513_b200 import cwb
    c = S.CONFIGS["R1"]
    ds = S.make(c)
    X = torch.as_tensor(ds.X, device=devname)
    Y = torch.as_tensor(ds.Y, device=devname)
    cfg = cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots, degree=c.degree,
                     df=c.df, batch_hint=c.B)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=devname)

    def ev(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    def step():
        p = cwb.Pool(X, cfg)
        p.train(Y, nu=c.nu, M=c.M)
        p.close()
    for _ in range(warmup):
        step()
    ts = []
    for i in range(steps):
        flush.fill_(i & 255)
        ts.append(ev(step))
    p = cwb.Pool(X, cfg)
    p.train(Y, nu=c.nu, M=c.M)
    ks = []
    for i in range(10):
        flush.fill_(i & 255)
        l0 = p.launches()
        ks.append(ev(lambda: p.train(Y, nu=c.nu, M=c.M)))
        nl = p.launches() - l0
    p.status()
    n_star = p.n_star
    p.close()
    ms, kms = float(np.mean(ts)), float(np.mean(ks))
    roof = sec8d_roofline(c.K, c.n, c.B, n_star, peaks, kms * 1e-3, c.M, "k_train_fused", bytes_extra=c.n * c.B * 8)
    return {"workload": "R1", "ms_per_step": ms, "value": c.K * c.n * c.B * c.M / (ms * 1e-3), "unit": UNIT,
            "iters_per_s": c.M / (ms * 1e-3), "kernel_ms": kms, "launches_per_call": int(nl),
            "roofline": {k: roof[k] for k in ("bound", "kernel", "achieved", "peak", "unit", "frac", "terms")}}


def findbest_b1(devname, peaks, name="R3", calls=15):
    """SURVEY Sec. 8(d) target: one findBestBaselearner (cwb_find_best) on ONE residual column at R3
    (u16 index vectors) against the HBM roofline of its algorithmic bytes K*n*2 + n*8.  L2 is flushed
    (256 MiB write) before every call and each call is timed alone with CUDA events; median."""
    import torch
    from paper_2110_03513_b200 import cwb
    c = S.CONFIGS[name]
    ds = S.make(c, reps=[0])
    X = torch.as_tensor(ds.X, device=devname)
    R = torch.as_tensor(ds.Y - ds.Y.mean(1, keepdims=True), device=devname)
    pool = cwb.Pool(X, cwb.Config(n_star_rule=c.n_star_rule, n_star_fixed=c.n_star_fixed, n_knots=c.n_knots,
                                  degree=c.degree, df=c.df))
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=devname)
    for _ in range(3):
        pool.find_best(R)
    ts = []
    for i in range(calls):
        buf.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pool.find_best(R)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    pool.status()
    pool.close()
    us = float(np.median(ts))
    alg = c.K * c.n * (1 if pool.n_star <= 256 else 2) + c.n * 8
    peak = float(peaks.get("hbm_gbs", 6548.2))
    return {"workload": name, "B": 1, "us": us, "alg_bytes": alg, "achieved_gbs": alg / us * 1e-3,
            "peak_gbs": peak, "frac": alg / us * 1e-3 / peak, "target_frac": 0.6,
            "kernels": "k_h1_stream + k_fit_narrow", "l2": "flushed before every call"}


def gram_path(X, Y, cfg, gcfg, flush, stream, peaks, args, direct_ms):
    """The cross-Gram formulation (cwb_set_path 3), timed like the headline step (fresh pool:
    cwb_init + cwb_train with the cross-Gram build, CUDA events, L2 flushed between steps) and reported
    separately -- never mixed into the direct path's numbers.  Phases from pools with the cross Gram cached:
    theta^[0] (one binMatVec pass, M = 0) and the M iterations (k_gram_train)."""
    import torch
    from paper_2110_03513_b200 import cwb
    K, n, B, M = cfg.K, cfg.n, cfg.B, cfg.M

    def ev(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    def step():
        p = cwb.Pool(X, gcfg)
        p.set_path(3)
        p.train(Y, nu=cfg.nu, M=M)
        p.close()
    for i in range(args.warmup):
        step()
    ts = []
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(float(i))
        ts.append(ev(step))
    # median: a fresh pool re-allocates the row-chunk basis buffer (1.3 GB at R3), and one of a few steps can
    # take an allocator stall (seen once under torchrun: 0.6 s); the mean is reported beside it
    ms = float(np.median(ts))
    ms_mean = float(np.mean(ts))
    p = cwb.Pool(X, gcfg)
    p.set_path(3)
    t_first0 = ev(lambda: p.train(Y, nu=cfg.nu, M=0))          # cross Gram + W + theta^[0]
    t_m0 = min(ev(lambda: p.train(Y, nu=cfg.nu, M=0)) for _ in range(3))   # theta^[0] only
    t_mm = min(ev(lambda: p.train(Y, nu=cfg.nu, M=M)) for _ in range(3))
    p.status()
    p_d = p.d
    p.close()
    t_x = t_first0 - t_m0
    t_it = t_mm - t_m0
    # dominant phase = the cross-Gram build through the joint bin counts of the K (K - 1) / 2 learner pairs
    # (k_idx_rowmajor, k_gram_pregather, k_gram_joint): per pair n integer increments
    # (u32 shared-memory atomics) and 6 n bytes of index traffic (the permuted index row read from the
    # row-major copy, written once, streamed once by the count pass); the contraction is O(n* d W) per pair
    pairs = K * (K - 1) // 2
    counts = pairs * n
    bytes_x = 6.0 * pairs * n
    n_sms = torch.cuda.get_device_properties(0).multi_processor_count
    sm_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    atoms_rate = 8.54 * n_sms * sm_hz   # measured u32 ATOMS.ADD rate, random of 1000 bins (profiles/r2h_ubench_atoms.txt)
    hbm = float(peaks["hbm_gbs"]) * 1e9
    t_atoms, t_hbm = counts / atoms_rate, bytes_x / hbm
    return {"path": "cross-Gram (cwb_set_path 3): s_k -= nu Z_k^T Z_k* theta*, exact reformulation of Alg. 1 for "
                    "L2 loss; parity tests/test_gpu_gram.py (R0-R3 vs the oracle, tie rule 1e-12)",
            "ms_per_step": ms, "ms_per_step_mean": ms_mean, "steps_timed": len(ts),
            "value": K * n * B * M / (ms * 1e-3), "unit": UNIT,
            "speedup_vs_direct": direct_ms / ms,
            "phases_ms": {"xgram_build": t_x, "theta0_binmatvec": t_m0, "iterations": t_it,
                          "iteration_us": t_it / max(M, 1) * 1e3},
            "roofline": {"kernel": "cross-Gram build (k_gram_pregather + k_gram_joint: joint bin counts of learner pairs)",
                         "bound": "hbm" if t_hbm >= t_atoms else "alu", "counts": counts, "bytes": bytes_x,
                         "t_atoms_ms": t_atoms * 1e3, "t_hbm_ms": t_hbm * 1e3, "t_kernel_ms": t_x,
                         "achieved": bytes_x / (t_x * 1e-3) / 1e9, "peak": hbm / 1e9, "unit": "GB/s",
                         "frac": max(t_atoms, t_hbm) / (t_x * 1e-3),
                         "note": "time from the difference of a fresh and a cached pool (M = 0); roofline time = "
                                 "max(index bytes / HBM, increments / measured u32 shared-atomic rate)"}}


def workload_config(c, n_star, d):
    return {"workload": c.name, "n": c.n, "K": c.K, "B_per_gpu": c.B, "M": c.M, "nu": c.nu,
            "n_star": n_star, "d": d, "df": c.df, "degree": c.degree, "n_knots": c.n_knots,
            "step": "cwb_init + cwb_train (all M iterations for B replications)",
            "l2": "flushed between steps (256 MiB write), flush outside the timed events"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="R3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", type=int, default=0, help="0 auto, 1 fused, 2 general")
    ap.add_argument("--algo", default="cwb", choices=["cwb", "acwb", "hcwb", "bernoulli"],
                    help="cwb: Alg. 1 supp. (default, the headline); acwb: Alg. 2; hcwb: Alg. 3; "
                         "bernoulli: Alg. 1 with the Bernoulli loss on seeded 0/1 targets")
    ap.add_argument("--shard", default="replications", choices=["replications", "rows", "learners"],
                    help="multi-GPU sharding: replications (weak, default), rows or learners (strong, one "
                         "collective per iteration)")
    ap.add_argument("--unbinned", action="store_true",
                    help="unbinned learners on the raw x (SURVEY NEXT-3): the baseline binning is compared to")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gram", action="store_true", help="skip the separately reported cross-Gram path (path 3)")
    ap.add_argument("--no-findbest", action="store_true",
                    help="skip the auxiliary B = 1 findBest measurement at R3 (SURVEY Sec. 8(d) target)")
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="training seconds of one reference-arm step (the sample of replications is sized to it)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference" or os.environ.get("BENCH_ALLOW_SHORT"), \
        "timing rules: at least 3 warm-up steps"
    cfg = S.CONFIGS[args.config]

    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    from paper_2110_03513_b200 import dist as D
    w = D.world_from_env()
    ws, rank, local = w.size, w.rank, w.local_rank
    torch.cuda.set_device(local)
    devname = f"cuda:{local}"
    if ws > 1:  # NCCL's communicator lines (stderr) let a scaling run verify nranks and the transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
    D.init_process_group(w, "nccl", torch.device(devname))
    from paper_2110_03513_b200 import cwb

    rows = args.shard == "rows"
    strong = args.shard in ("rows", "learners")
    if strong and args.algo != "cwb":
        raise SystemExit("--shard rows / learners support --algo cwb only")
    # replications: this rank's block (weak scaling), rank r owns [r*B, (r+1)*B);
    # rows: the workload's B replications on every rank, this rank's row block of them;
    # learners: the workload's B replications and rows on every rank, this rank's block of learners
    reps = range(cfg.B) if strong else D.replication_block(cfg.B, rank)
    ds = S.make(cfg, reps=reps)
    blk = D.row_block(cfg.n, rank, ws) if rows else range(cfg.n)
    X = torch.as_tensor(ds.X, device=devname)
    Ysrc = S.binary_targets(ds) if args.algo == "bernoulli" else ds.Y
    Y_host = np.ascontiguousarray(Ysrc[:, blk.start:blk.stop])
    Y = torch.as_tensor(Y_host, device=devname)
    gcfg = cwb.Config(n_star_rule=cfg.n_star_rule, n_star_fixed=cfg.n_star_fixed, n_knots=cfg.n_knots,
                      degree=cfg.degree, df=cfg.df, batch_hint=0 if strong or args.unbinned else cfg.B,
                      unbinned=int(args.unbinned),
                      train_hint={"cwb": 0, "acwb": 1, "hcwb": 2, "bernoulli": 3}[args.algo])
    comm = None
    if strong:  # libcwb's own NCCL communicator, id from rank 0 over the torch process group
        uid = D.nccl_unique_id(w, torch.device(devname)) if ws > 1 else cwb.cwb_comm_unique_id()
        comm = cwb.Comm(rank, ws, unique_id=uid)

    def new_pool(Xsrc):
        p_ = cwb.Pool(Xsrc, gcfg)
        if comm is not None:
            if rows:
                p_.attach(comm)
            else:
                p_.attach_learners(comm)
        return p_
    B, K, n, M = cfg.B, cfg.K, cfg.n, cfg.M
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=devname)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps + args.warmup)]
    outs = None
    launches = []
    vm = torch.as_tensor(S.validation_mask(n), device=devname) if args.algo == "hcwb" else None

    def train(pool, out=None):
        if args.algo == "acwb":   # Alg. 2, gamma = 0.0034
            return pool.train_acwb(Y, nu=cfg.nu, gamma=0.0034, M=M)
        if args.algo == "hcwb":   # Alg. 3, gamma = 0.037, pat0 = 5, 30 % validation
            return pool.train_hcwb(Y, vm, nu=cfg.nu, gamma=0.037, pat0=5, M=M)
        if args.algo == "bernoulli":  # Alg. 1, Bernoulli loss
            return pool.train_bernoulli(Y, nu=cfg.nu, M=M)
        return pool.train(Y, nu=cfg.nu, M=M, out=out)

    def step(i):
        nonlocal outs
        a, b, c_ = ev[i]
        a.record(stream)
        pool = new_pool(X)
        if args.path:
            pool.set_path(args.path)
        b.record(stream)
        outs = train(pool, outs)
        if ws > 1 and not strong and args.algo == "cwb":  # one all-gather of the results
            D.gather_results(outs, w)
        c_.record(stream)
        launches.append(pool.launches())
        pool.close()

    for i in range(args.warmup):
        step(i)
        flush.fill_(float(i))
    torch.cuda.synchronize()
    pool = cwb.Pool(X, gcfg)
    pool.status()
    n_star, d = pool.n_star, pool.d
    pool.close()

    def barrier():
        D.barrier(w)
        torch.cuda.synchronize()

    launches.clear()
    clk = ClockSampler(local)
    barrier()
    with clk:
        for i in range(args.warmup, args.warmup + args.steps):
            flush.fill_(float(i))
            step(i)
        barrier()
    step_ms = np.array([ev[i][0].elapsed_time(ev[i][2]) for i in range(args.warmup, args.warmup + args.steps)])
    train_ms = np.array([ev[i][1].elapsed_time(ev[i][2]) for i in range(args.warmup, args.warmup + args.steps)])
    init_ms = step_ms - train_ms
    total_ms = D.max_over_ranks(float(step_ms.sum()), w, devname)
    ms_per_step = total_ms / args.steps
    # learner-row evaluations per step: K*n*B per findBest; ACWB fits twice per
    # iteration; HCWB twice while accelerated (its switch iterations from the last step), then once
    if args.algo == "acwb":
        evals_rank = 2 * K * n * B * M
    elif args.algo == "hcwb":
        sw = outs["switch_iter"].cpu().numpy().astype(np.int64)
        evals_rank = int(K * n * (2 * sw + (M - sw)).sum())
    else:
        evals_rank = K * n * B * M
    evals = evals_rank if strong else evals_rank * ws
    value = evals / (ms_per_step * 1e-3)

    # ---- end-to-end through the host-pointer C-ABI call (pinned host buffers)
    Xh = torch.as_tensor(ds.X).pin_memory()
    Yh = torch.as_tensor(Y_host).pin_memory()
    outh = {"offset": torch.empty(B, dtype=torch.float64).pin_memory(),
            "theta_agg": torch.empty((B, K, d), dtype=torch.float64).pin_memory(),
            "k_trace": torch.empty((M, B), dtype=torch.int32).pin_memory(),
            "sse_trace": torch.empty((M, B), dtype=torch.float64).pin_memory(),
            "risk_trace": torch.empty((M, B), dtype=torch.float64).pin_memory()}
    lib = cwb.load()
    import ctypes as C
    ccfg = gcfg.c()
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def e2e_step():
        rc = lib.cwb_fit_host(P(Xh), n, K, C.byref(ccfg), P(Yh), B, float(cfg.nu), M, P(outh["offset"]),
                              P(outh["theta_agg"]), P(outh["k_trace"]), P(outh["sse_trace"]),
                              P(outh["risk_trace"]), C.c_void_p(stream.cuda_stream))
        if rc:
            raise cwb.CwbError(rc, lib.cwb_last_error(None).decode())

    if args.algo != "cwb" or strong:
        Xd = torch.empty_like(X)
        Yd = torch.empty_like(Y)
        host_out = {}

        def e2e_step():  # noqa: F811 - pinned H2D of X, Y; pool + train; D2H of every output
            Xd.copy_(Xh, non_blocking=True)
            Yd.copy_(Yh, non_blocking=True)
            pool = new_pool(Xd)
            if args.algo == "cwb":
                o = pool.train(Yd, nu=cfg.nu, M=M)
            elif args.algo == "acwb":
                o = pool.train_acwb(Yd, nu=cfg.nu, gamma=0.0034, M=M)
            elif args.algo == "bernoulli":
                o = pool.train_bernoulli(Yd, nu=cfg.nu, M=M)
            else:
                o = pool.train_hcwb(Yd, vm, nu=cfg.nu, gamma=0.037, pat0=5, M=M)
            for k_, v_ in o.items():
                if k_ not in host_out:
                    host_out[k_] = torch.empty(v_.shape, dtype=v_.dtype).pin_memory()
                host_out[k_].copy_(v_, non_blocking=True)
            pool.close()
            stream.synchronize()
    for i in range(3):
        e2e_step()
    e_ms = []
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        e1.synchronize()
        e_ms.append(e0.elapsed_time(e1))
    e2e_ms = D.max_over_ranks(float(np.mean(e_ms)), w, devname)
    h2d = ds.X.nbytes + Y_host.nbytes
    d2h = sum(v.numel() * v.element_size() for v in (outh if args.algo == "cwb" and not strong else host_out).values())

    # ---- kernel-only time of the dominant kernel, CUDA events on the launching stream, same launch
    #      configuration as the step: the whole k_train_fused launch when cwb_train is one persistent launch
    #      (plan cached), else the binMatVec phase H1 of the per-iteration path (libcwb brackets its launches
    #      with events: cwb_set_h1_timing / cwb_get_h1_time)
    kpool = new_pool(X)
    if args.path:
        kpool.set_path(args.path)
    kouts = train(kpool)
    kpool.status()
    k_ms, h1_ms, h1_n = [], 0.0, 0
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = kpool.launches()
        kpool.set_h1_timing(True)
        e0.record(stream)
        kouts = train(kpool, kouts)
        e1.record(stream)
        e1.synchronize()
        t_, n_ = kpool.h1_time()
        h1_ms += t_
        h1_n += n_
        k_ms.append(e0.elapsed_time(e1))
        k_launches = kpool.launches() - l0
    kpool.set_h1_timing(False)
    kpool.close()
    kernel_ms = float(np.median(k_ms))  # median: one allocator stall in ten calls once tripled the mean (HCWB, r2k)
    if rank == 0:
        peaks, src = load_peaks()
        n_loc = len(blk)
        fits = 1 if args.algo in ("cwb", "bernoulli") else 2
        sm_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        n_sms = torch.cuda.get_device_properties(devname).multi_processor_count
        if k_launches == 1:   # one persistent launch: M iterations of H1-H6 on chip
            roof = sec8d_roofline(K, n_loc, B * fits, n_star, peaks, kernel_ms * 1e-3, M,
                                  f"k_train_fused ({args.algo} mode)" if args.algo != "cwb" else "k_train_fused",
                                  bytes_extra=n_loc * B * fits * 8)
            roof["units"] = f"{M} iterations per launch (bytes_alg per iteration = K n idx + 2 n B 8)"
        elif h1_n > 0:        # per-iteration kernels: the binMatVec phase H1 dominates the iteration
            roof = sec8d_roofline(K, n_loc, B * fits, n_star, peaks, h1_ms / h1_n * 1e-3, 1,
                                  "H1 binMatVec (k_h1, or the k_h1c row-chunk launches) of one iteration")
            roof["units"] = f"one H1 phase (mean of {h1_n} timed phases); bytes_alg = K n idx + n B 8"
            roof["h1_share_of_train"] = (h1_ms / (len(k_ms))) / kernel_ms
            # the binding on-chip unit: each (learner, row, column) add reads 8 B of the residual block
            # from L2 (the 32-column tile of R fits L2 at R3; chunked at R4)
            l2b = 8.0 * K * n_loc * B * fits
            l2 = float(peaks.get("l2_read_gbs", 0.0))
            roof["l2_gather"] = {"bytes_per_phase": l2b, "achieved_gbs": l2b / (h1_ms / h1_n * 1e-3) / 1e9,
                                 "peak_gbs": l2 or None, "frac": (l2b / (h1_ms / h1_n * 1e-3) / 1e9 / l2) if l2 else None,
                                 "note": "measured L2-resident read bandwidth, profiles/peaks_fp64.json"}
        else:
            roof = sec8d_roofline(K, n_loc, B * fits, n_star, peaks, kernel_ms * 1e-3, M,
                                  f"{args.algo} per-iteration kernels (whole cwb_train call)",
                                  bytes_extra=n_loc * B * fits * 8)
        # iteration level: M x max(bytes/HBM, adds/DADD) against the measured cwb_train time
        it = sec8d_roofline(K, n_loc, B * fits, n_star, peaks, kernel_ms * 1e-3, M, "cwb_train (all kernels)",
                            bytes_extra=n_loc * B * fits * 8)
        roof["train_frac"] = it["frac"]
        roof["train_ms"] = kernel_ms
        roof["launches_per_call"] = int(k_launches)
        roof["peak_src"] = {"hbm": f"MEASURED_PEAKS.json hbm_gbs ({src})", "dadd": peaks.get("fp64_src")}
        traffic = None
        smem_wf = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                tj = json.load(open(tp))
                if args.algo == "cwb" and not strong and not args.unbinned:  # ncu --set full of the same kernel
                    key = cfg.name if k_launches == 1 else cfg.name + "_h1"
                    traffic = tj.get(key)
                    smem_wf = tj.get("smem_wavefronts", {}).get(key)
            except Exception:
                traffic = None
        roof["traffic"] = traffic
        if k_launches == 1:
            rb = 2 if B > n_sms else 1  # replications per CTA
            ctas_per_sm = -(-(-(-B // rb)) // n_sms)
            roof["smem_pipe_frac"] = smem_wf / (kernel_ms * 1e-3 * sm_hz * n_sms) if smem_wf else None
            roof["smem_gather_ceiling"] = {
                "h1_floor_ms": K * n * ctas_per_sm * M / (GATHER_LANE_LOADS_PER_CLK[rb] * sm_hz) * 1e3,
                "note": ("time H1 alone would take at the measured conflict-free shared-memory gather rate "
                         "(profiles/ubench_smem_gather.txt); the binding on-chip ceiling of this kernel")}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (paper Sec. 4.1.1 generator, seeded; OpenML sets not available)",
            "config": dict(workload_config(cfg, n_star, d), algo=args.algo, shard=args.shard,
                           learners="unbinned" if args.unbinned else "binned",
                           parallelism=(f"{args.shard}{ws}")),
            "iters_per_s": M / (ms_per_step * 1e-3),
            "phase_ms": {"init": float(np.mean(init_ms)), "train": float(np.mean(train_ms))},
            "roofline": roof,
            "e2e": {"value": evals / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
                    "api": ("cwb_fit_host (pinned host buffers, copies + init + train + sync)"
                            if args.algo == "cwb" and not strong
                            else f"pinned H2D of X, Y + cwb_init + cwb_train_{args.algo} + D2H of all outputs")},
            "clocks": clk.summary(),
            "gpu_launches": int(sum(launches)),
        }
        if args.algo == "cwb" and not strong and not args.unbinned and ws == 1 and not args.no_findbest:
            if cfg.name != "R1":
                try:
                    line["r1"] = r1_rung(devname, peaks)
                except Exception as e:
                    line["r1"] = {"error": str(e)}
            for fb_cfg in ("R3", "R4"):
                try:  # after the timed region: does not touch the step measurement
                    line[f"findbest_b1_{fb_cfg}"] = findbest_b1(devname, peaks, fb_cfg)
                except Exception as e:
                    line[f"findbest_b1_{fb_cfg}"] = {"error": str(e)}
        if args.algo == "cwb" and not strong and not args.unbinned and ws == 1 and not args.no_gram:
            try:  # after the timed region: the separately reported cross-Gram path (cwb_set_path 3)
                line["gram"] = gram_path(X, Y, cfg, gcfg, flush, stream, peaks, args, ms_per_step)
            except Exception as e:
                line["gram"] = {"error": str(e)}
        if not args.no_cpu_baseline and ws == 1:
            try:
                line["cpu_baseline"] = {k: v for k, v in oracle_sample(cfg, algo=args.algo,
                                                                        unbinned=args.unbinned).items()
                                        if k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as e:  # keep the GPU line even if the host leg fails
                line["cpu_baseline"] = {"error": str(e)}
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
