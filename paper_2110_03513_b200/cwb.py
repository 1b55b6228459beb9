"""Thin Python binding of include/cwb.h (argument marshalling only).

Every function here has the name of the C entry point it calls and does no
arithmetic of the method: it checks dtypes/shapes, allocates outputs with
torch on the tensors' device, passes raw device pointers and the current
CUDA stream, and raises CwbError on a non-zero status.  There is no CPU or
PyTorch fallback: if libcwb.so is missing, load() raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
# CWB_LIB selects another in-tree build of the same sources (tests: libcwb_jitter.so)
LIB_PATH = os.environ.get("CWB_LIB") or os.path.join(HERE, "libcwb.so")

CODES = {0: "CWB_OK", -1: "CWB_EINVAL", -2: "CWB_EDEGENERATE", -3: "CWB_ECALIB", -4: "CWB_ENONFINITE",
         -5: "CWB_EEMPTY", -6: "CWB_ECUDA", -7: "CWB_ENCCL", -8: "CWB_ENOMEM", -9: "CWB_EUNSUPPORTED"}

# the exported symbols declared in include/cwb.h
SYMBOLS = ["cwb_default_config", "cwb_version", "cwb_bin", "cwb_bin_mat_mat", "cwb_bin_mat_vec",
           "cwb_init", "cwb_status", "cwb_last_error", "cwb_get_dims", "cwb_get_lambda", "cwb_get_n_star_k", "cwb_get_pool",
           "cwb_set_path", "cwb_set_narrow", "cwb_find_best", "cwb_train", "cwb_train_bernoulli", "cwb_train_folds", "cwb_train_acwb", "cwb_train_hcwb", "cwb_fit_host", "cwb_predict",
           "cwb_launch_count", "cwb_set_phase_timing", "cwb_set_h1_timing", "cwb_get_h1_time", "cwb_free", "cwb_comm_unique_id", "cwb_comm_init",
           "cwb_comm_init_fn", "cwb_comm_free", "cwb_attach_comm", "cwb_attach_comm_learners", "cwb_get_rows"]


class CwbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{CODES.get(code, code)}: {msg}")
        self.code = code
        self.name = CODES.get(code, str(code))


class cwb_config(C.Structure):
    _fields_ = [("n_star_rule", C.c_int32), ("n_star_fixed", C.c_int32), ("degree", C.c_int32),
                ("n_knots", C.c_int32), ("df", C.c_double), ("df_kind", C.c_int32), ("batch_hint", C.c_int32),
                ("unbinned", C.c_int32), ("train_hint", C.c_int32)]


@dataclass
class Config:
    n_star_rule: int = 0
    n_star_fixed: int = 0
    degree: int = 3
    n_knots: int = 20
    df: float = 5.0
    df_kind: int = 1
    batch_hint: int = 0  # expected B of the train calls: lets cwb_init pre-build the fused plan
    unbinned: int = 0    # 1: learners on the raw x (no binning), SURVEY NEXT-3
    train_hint: int = 0  # the training call batch_hint is for: 0 cwb, 1 acwb, 2 hcwb, 3 bernoulli

    def c(self) -> cwb_config:
        return cwb_config(self.n_star_rule, self.n_star_fixed, self.degree, self.n_knots, self.df,
                          self.df_kind, self.batch_hint, self.unbinned, self.train_hint)


_lib = None
_vp, _i32, _i64, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
# int (*cwb_allreduce_fn)(double* buf, int64_t count, cudaStream_t stream, void* user)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


def load() -> C.CDLL:
    """Load libcwb.so (built by build.py / __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2110_03513_b200.build` "
                          "(the engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.cwb_default_config.argtypes = [C.POINTER(cwb_config)]
    L.cwb_default_config.restype = None
    L.cwb_version.restype = C.c_int
    L.cwb_bin.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _vp]
    L.cwb_bin_mat_mat.argtypes = [_vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, _vp]
    L.cwb_bin_mat_vec.argtypes = [_vp, _i32, _i32, _vp, _i32, _vp, _vp, _i64, _i32, _vp, _vp]
    L.cwb_init.argtypes = [C.POINTER(_vp), _vp, _i64, _i32, C.POINTER(cwb_config), _vp]
    L.cwb_status.argtypes = [_vp]
    L.cwb_last_error.argtypes = [_vp]
    L.cwb_last_error.restype = C.c_char_p
    L.cwb_get_dims.argtypes = [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i64)]
    L.cwb_get_lambda.argtypes = [_vp, _vp]
    L.cwb_get_n_star_k.argtypes = [_vp, _vp]
    L.cwb_get_pool.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
    L.cwb_set_path.argtypes = [_vp, _i32]
    L.cwb_set_narrow.argtypes = [_vp, _i32]
    L.cwb_find_best.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _vp]
    L.cwb_train.argtypes = [_vp, _vp, _i32, _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
    L.cwb_train_bernoulli.argtypes = [_vp, _vp, _i32, _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
    L.cwb_train_folds.argtypes = [_vp, _vp, _i32, _vp, _i32, _vp, _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.cwb_train_acwb.argtypes = [_vp, _vp, _i32, _f64, _f64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.cwb_train_hcwb.argtypes = [_vp, _vp, _i32, _vp, _f64, _f64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp]
    L.cwb_fit_host.argtypes = [_vp, _i64, _i32, C.POINTER(cwb_config), _vp, _i32, _f64, _i32,
                               _vp, _vp, _vp, _vp, _vp, _vp]
    L.cwb_predict.argtypes = [_vp, _vp, _i64, _vp, _vp, _i32, _vp, _vp]
    L.cwb_set_phase_timing.argtypes = [_vp, _vp]
    L.cwb_set_h1_timing.argtypes = [_vp, _i32]
    L.cwb_get_h1_time.argtypes = [_vp, C.POINTER(_f64), C.POINTER(_i32)]
    L.cwb_launch_count.argtypes = [_vp]
    L.cwb_launch_count.restype = C.c_int64
    L.cwb_free.argtypes = [_vp]
    L.cwb_free.restype = None
    L.cwb_comm_unique_id.argtypes = [_vp]
    L.cwb_comm_init.argtypes = [C.POINTER(_vp), _vp, _i32, _i32]
    L.cwb_comm_init_fn.argtypes = [C.POINTER(_vp), ALLREDUCE_FN, _vp, _i32, _i32]
    L.cwb_comm_free.argtypes = [_vp]
    L.cwb_comm_free.restype = None
    L.cwb_attach_comm.argtypes = [_vp, _vp]
    L.cwb_attach_comm_learners.argtypes = [_vp, _vp]
    L.cwb_get_rows.argtypes = [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i32)]
    _lib = L
    return L


def _chk(code: int, ctx=None) -> None:
    if code != 0:
        msg = load().cwb_last_error(ctx)
        raise CwbError(code, msg.decode() if msg else "")


def _stream(t=None) -> int:
    import torch
    dev = t.device if t is not None else torch.device("cuda")
    return torch.cuda.current_stream(dev).cuda_stream


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev_f64(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError(f"{name} must be a float64 CUDA tensor")
    return t.contiguous()


def _idx_bytes(idx):
    import torch
    if idx.dtype == torch.uint8:
        return 1
    if idx.dtype == torch.uint16:
        return 2
    raise TypeError("idx must be uint8 or uint16")


# ------------------------------------------------------------------ primitives

def cwb_bin(x, n_star: int, idx_bytes: int | None = None):
    """P:L859-861 -> (z, bnd, idx) on x.device."""
    import torch
    x = _dev_f64(x, "x")
    if idx_bytes is None:
        idx_bytes = 1 if n_star <= 256 else 2
    z = torch.empty(n_star, dtype=torch.float64, device=x.device)
    bnd = torch.empty(max(n_star - 1, 1), dtype=torch.float64, device=x.device)
    idx = torch.empty(x.numel(), dtype=torch.uint8 if idx_bytes == 1 else torch.uint16, device=x.device)
    _chk(load().cwb_bin(_ptr(x), x.numel(), n_star, _ptr(z), _ptr(bnd), _ptr(idx), idx_bytes, _stream(x)))
    return z, bnd[: n_star - 1], idx


def cwb_bin_mat_mat(Zb, idx, w=None):
    """Algorithm binMatMat: Zb^T diag(c) Zb."""
    import torch
    Zb = _dev_f64(Zb, "Zb")
    ns, d = Zb.shape
    w = None if w is None else _dev_f64(w, "w")
    out = torch.empty((d, d), dtype=torch.float64, device=Zb.device)
    _chk(load().cwb_bin_mat_mat(_ptr(Zb), ns, d, _ptr(idx.contiguous()), _idx_bytes(idx), _ptr(w),
                                idx.numel(), _ptr(out), _stream(Zb)))
    return out


def cwb_bin_mat_vec(Zb, idx, R, w=None):
    """Algorithm binMatVec for R[B][n] -> out[B][d]."""
    import torch
    Zb = _dev_f64(Zb, "Zb")
    R = _dev_f64(R, "R")
    if R.dim() == 1:
        R = R[None]
    ns, d = Zb.shape
    B, n = R.shape
    w = None if w is None else _dev_f64(w, "w")
    out = torch.empty((B, d), dtype=torch.float64, device=Zb.device)
    _chk(load().cwb_bin_mat_vec(_ptr(Zb), ns, d, _ptr(idx.contiguous()), _idx_bytes(idx), _ptr(w),
                                _ptr(R), n, B, _ptr(out), _stream(Zb)))
    return out


# ------------------------------------------------------------------- context

def cwb_init(X, cfg: Config | None = None):
    """Build the base-learner pool on X[K][n] (device).  Returns a context handle."""
    X = _dev_f64(X, "X")
    K, n = X.shape
    h = C.c_void_p()
    c = (cfg or Config()).c()
    _chk(load().cwb_init(C.byref(h), _ptr(X), n, K, C.byref(c), _stream(X)))
    return h


def cwb_status(ctx) -> None:
    _chk(load().cwb_status(ctx), ctx)


def cwb_get_dims(ctx):
    ns, d, K, n = _i32(), _i32(), _i32(), _i64()
    _chk(load().cwb_get_dims(ctx, C.byref(ns), C.byref(d), C.byref(K), C.byref(n)), ctx)
    return ns.value, d.value, K.value, n.value


def cwb_get_lambda(ctx):
    import numpy as np
    ns, d, K, n = cwb_get_dims(ctx)
    out = np.empty(K, dtype=np.float64)
    _chk(load().cwb_get_lambda(ctx, out.ctypes.data_as(C.c_void_p)), ctx)
    return out


def cwb_get_n_star_k(ctx):
    import numpy as np
    ns, d, K, n = cwb_get_dims(ctx)
    out = np.empty(K, dtype=np.int32)
    _chk(load().cwb_get_n_star_k(ctx, out.ctypes.data_as(C.c_void_p)), ctx)
    return out


def cwb_get_pool(ctx, device="cuda"):
    import torch
    ns, d, K, n = cwb_get_dims(ctx)
    f = dict(dtype=torch.float64, device=device)
    z = torch.empty((K, ns), **f)
    idx = torch.empty((K, n), dtype=torch.uint16, device=device)
    Zb = torch.empty((K, ns, d), **f)
    G = torch.empty((K, d, d), **f)
    Ainv = torch.empty((K, d, d), **f)
    _chk(load().cwb_get_pool(ctx, _ptr(z), _ptr(idx), _ptr(Zb), _ptr(G), _ptr(Ainv)), ctx)
    return dict(z=z, idx=idx, Zb=Zb, G=G, Ainv=Ainv)


def cwb_set_path(ctx, path: int) -> None:
    _chk(load().cwb_set_path(ctx, path), ctx)


def cwb_set_narrow(ctx, mode: int) -> None:
    _chk(load().cwb_set_narrow(ctx, mode), ctx)


def cwb_find_best(ctx, R):
    """findBestBaselearner for R[B][n] -> (k[B], theta[B][d], sse[B])."""
    import torch
    R = _dev_f64(R, "R")
    if R.dim() == 1:
        R = R[None]
    ns, d, K, n = cwb_get_dims(ctx)
    B = R.shape[0]
    k = torch.empty(B, dtype=torch.int32, device=R.device)
    th = torch.empty((B, d), dtype=torch.float64, device=R.device)
    sse = torch.empty(B, dtype=torch.float64, device=R.device)
    _chk(load().cwb_find_best(ctx, _ptr(R), B, _ptr(k), _ptr(th), _ptr(sse), _stream(R)), ctx)
    return k, th, sse


def cwb_train(ctx, Y, nu: float = 0.05, M: int = 200, traces: bool = True, out=None):
    """Vanilla CWB (Alg. 1 supp.) for Y[B][n].  Returns a dict of device tensors."""
    import torch
    Y = _dev_f64(Y, "Y")
    ns, d, K, n = cwb_get_dims(ctx)
    B = Y.shape[0]
    if out is None:
        f = dict(dtype=torch.float64, device=Y.device)
        out = dict(offset=torch.empty(B, **f), theta_agg=torch.empty((B, K, d), **f))
        if traces:
            out.update(k_trace=torch.empty((M, B), dtype=torch.int32, device=Y.device),
                       sse_trace=torch.empty((M, B), **f), risk_trace=torch.empty((M, B), **f))
    _chk(load().cwb_train(ctx, _ptr(Y), B, float(nu), M, _ptr(out["offset"]), _ptr(out["theta_agg"]),
                          _ptr(out.get("k_trace")), _ptr(out.get("sse_trace")),
                          _ptr(out.get("risk_trace")), _stream(Y)), ctx)
    return out


def cwb_train_bernoulli(ctx, Y, nu: float = 0.05, M: int = 200, traces: bool = True):
    """CWB with the Bernoulli loss (y in {0, 1}) for Y[B][n].  Returns a dict of device tensors."""
    import torch
    Y = _dev_f64(Y, "Y")
    ns, d, K, n = cwb_get_dims(ctx)
    B = Y.shape[0]
    f = dict(dtype=torch.float64, device=Y.device)
    out = dict(offset=torch.empty(B, **f), theta_agg=torch.empty((B, K, d), **f))
    if traces:
        out.update(k_trace=torch.empty((M, B), dtype=torch.int32, device=Y.device),
                   sse_trace=torch.empty((M, B), **f), risk_trace=torch.empty((M, B), **f))
    _chk(load().cwb_train_bernoulli(ctx, _ptr(Y), B, float(nu), M, _ptr(out["offset"]), _ptr(out["theta_agg"]),
                                    _ptr(out.get("k_trace")), _ptr(out.get("sse_trace")),
                                    _ptr(out.get("risk_trace")), _stream(Y)), ctx)
    return out


def cwb_train_folds(ctx, Y, fold_of_row, F: int, fold_of_rep, nu: float = 0.05, M: int = 200):
    """CWB with per-replication CV folds for Y[B][n]; fold_of_row uint8[n], fold_of_rep int32[B] (device)."""
    import torch
    Y = _dev_f64(Y, "Y")
    if fold_of_row.dtype != torch.uint8 or fold_of_rep.dtype != torch.int32:
        raise TypeError("fold_of_row must be uint8 and fold_of_rep int32")
    ns, d, K, n = cwb_get_dims(ctx)
    B = Y.shape[0]
    f = dict(dtype=torch.float64, device=Y.device)
    out = dict(offset=torch.empty(B, **f), theta_agg=torch.empty((B, K, d), **f),
               k_trace=torch.empty((M, B), dtype=torch.int32, device=Y.device),
               sse_trace=torch.empty((M, B), **f), risk_trace=torch.empty((M, B), **f),
               val_risk_trace=torch.empty((M, B), **f))
    _chk(load().cwb_train_folds(ctx, _ptr(Y), B, _ptr(fold_of_row.contiguous()), F, _ptr(fold_of_rep.contiguous()),
                                float(nu), M, _ptr(out["offset"]), _ptr(out["theta_agg"]), _ptr(out["k_trace"]),
                                _ptr(out["sse_trace"]), _ptr(out["risk_trace"]), _ptr(out["val_risk_trace"]),
                                _stream(Y)), ctx)
    return out


def cwb_train_acwb(ctx, Y, nu: float = 0.05, gamma: float = 0.0034, M: int = 200, traces: bool = True):
    """Accelerated CWB (Alg. 2) for Y[B][n].  Returns a dict of device tensors."""
    import torch
    Y = _dev_f64(Y, "Y")
    ns, d, K, n = cwb_get_dims(ctx)
    B = Y.shape[0]
    f = dict(dtype=torch.float64, device=Y.device)
    out = dict(offset=torch.empty(B, **f), theta_f=torch.empty((B, K, d), **f), theta_h=torch.empty((B, K, d), **f))
    if traces:
        out.update(k_trace=torch.empty((M, B), dtype=torch.int32, device=Y.device),
                   kcor_trace=torch.empty((M, B), dtype=torch.int32, device=Y.device),
                   sse_trace=torch.empty((M, B), **f), risk_trace=torch.empty((M, B), **f))
    _chk(load().cwb_train_acwb(ctx, _ptr(Y), B, float(nu), float(gamma), M, _ptr(out["offset"]), _ptr(out["theta_f"]),
                               _ptr(out["theta_h"]), _ptr(out.get("k_trace")), _ptr(out.get("kcor_trace")),
                               _ptr(out.get("sse_trace")), _ptr(out.get("risk_trace")), _stream(Y)), ctx)
    return out


def cwb_train_hcwb(ctx, Y, val_mask, nu: float = 0.05, gamma: float = 0.037, pat0: int = 5, M: int = 200):
    """Hybrid CWB (Alg. 3) for Y[B][n]; val_mask[n] uint8 (1 = validation row).  Dict of device tensors."""
    import torch
    Y = _dev_f64(Y, "Y")
    if not isinstance(val_mask, torch.Tensor) or val_mask.dtype != torch.uint8 or not val_mask.is_cuda:
        raise TypeError("val_mask must be a uint8 CUDA tensor")
    val_mask = val_mask.contiguous()
    ns, d, K, n = cwb_get_dims(ctx)
    B = Y.shape[0]
    f = dict(dtype=torch.float64, device=Y.device)
    i32 = dict(dtype=torch.int32, device=Y.device)
    out = dict(offset=torch.empty(B, **f), theta_f=torch.empty((B, K, d), **f),
               k_trace=torch.empty((M, B), **i32), kcor_trace=torch.empty((M, B), **i32),
               sse_trace=torch.empty((M, B), **f), risk_trace=torch.empty((M, B), **f),
               val_risk_trace=torch.empty((M, B), **f), switch_iter=torch.empty(B, **i32))
    _chk(load().cwb_train_hcwb(ctx, _ptr(Y), B, _ptr(val_mask), float(nu), float(gamma), int(pat0), M,
                               _ptr(out["offset"]), _ptr(out["theta_f"]), _ptr(out["k_trace"]),
                               _ptr(out["kcor_trace"]), _ptr(out["sse_trace"]), _ptr(out["risk_trace"]),
                               _ptr(out["val_risk_trace"]), _ptr(out["switch_iter"]), _stream(Y)), ctx)
    return out


def cwb_fit_host(X, Y, cfg: Config | None = None, nu: float = 0.05, M: int = 200, stream=None):
    """Whole fit from HOST numpy arrays (copies inside the call)."""
    import numpy as np
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    K, n = X.shape
    B = Y.shape[0]
    c = (cfg or Config()).c()
    d = c.n_knots + c.degree + 1
    off = np.empty(B)
    agg = np.empty((B, K, d))
    kt = np.empty((M, B), dtype=np.int32)
    st = np.empty((M, B))
    rt = np.empty((M, B))
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    _chk(load().cwb_fit_host(p(X), n, K, C.byref(c), p(Y), B, float(nu), M, p(off), p(agg), p(kt), p(st),
                             p(rt), stream))
    return dict(offset=off, theta_agg=agg, k_trace=kt, sse_trace=st, risk_trace=rt)


def cwb_predict(ctx, Xnew, offset, theta_agg):
    import torch
    Xnew = _dev_f64(Xnew, "Xnew")
    offset = _dev_f64(offset, "offset")
    theta_agg = _dev_f64(theta_agg, "theta_agg")
    K, m = Xnew.shape
    B = offset.numel()
    out = torch.empty((B, m), dtype=torch.float64, device=Xnew.device)
    _chk(load().cwb_predict(ctx, _ptr(Xnew), m, _ptr(offset), _ptr(theta_agg), B, _ptr(out),
                            _stream(Xnew)), ctx)
    return out


def cwb_launch_count(ctx) -> int:
    return int(load().cwb_launch_count(ctx))


def cwb_set_phase_timing(ctx, cycles4=None) -> None:
    """cycles4: int64 CUDA tensor of 4 elements (or None to switch off)."""
    _chk(load().cwb_set_phase_timing(ctx, _ptr(cycles4)), ctx)


def cwb_set_h1_timing(ctx, on: bool) -> None:
    _chk(load().cwb_set_h1_timing(ctx, int(bool(on))), ctx)


def cwb_get_h1_time(ctx):
    """(summed milliseconds, number of bracketed H1 phases) since the last call; synchronises."""
    ms, np_ = _f64(0.0), _i32(0)
    _chk(load().cwb_get_h1_time(ctx, C.byref(ms), C.byref(np_)), ctx)
    return float(ms.value), int(np_.value)


def cwb_free(ctx) -> None:
    if ctx:
        load().cwb_free(ctx)


# ------------------------------------------------------------- row sharding

def cwb_comm_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (call on one rank, send the bytes to the others)."""
    buf = C.create_string_buffer(128)
    _chk(load().cwb_comm_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


class Comm:
    """RAII wrapper of a cwb_comm: an NCCL communicator built by libcwb (unique_id given), or
    the caller's collective fn(buf_ptr, count, stream_ptr) -> None, which must replace the
    device fp64 array buf[count] by its sum over the ranks (include/cwb.h)."""

    def __init__(self, rank: int, world: int, unique_id: bytes | None = None, fn=None):
        self.rank, self.world, self.h, self._cb = rank, world, C.c_void_p(), None
        if unique_id is not None:
            if len(unique_id) != 128:
                raise ValueError("unique_id must be 128 bytes")
            buf = C.create_string_buffer(bytes(unique_id), 128)
            _chk(load().cwb_comm_init(C.byref(self.h), C.cast(buf, C.c_void_p), rank, world))
        elif fn is not None:
            def tramp(buf, count, stream, user):
                try:
                    fn(buf, count, stream)
                    return 0
                except Exception:  # noqa: BLE001 -- reported to C as a failed collective
                    import traceback
                    traceback.print_exc()
                    return 1
            self._cb = ALLREDUCE_FN(tramp)
            _chk(load().cwb_comm_init_fn(C.byref(self.h), self._cb, None, rank, world))
        else:
            raise ValueError("need unique_id or fn")

    def close(self):
        if self.h:
            load().cwb_comm_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cwb_attach_comm(ctx, comm: Comm) -> None:
    """Row-shard ctx over comm (include/cwb.h "row sharding")."""
    _chk(load().cwb_attach_comm(ctx, comm.h), ctx)


def cwb_get_rows(ctx):
    """(row_begin, n_rows, rank, world) of the context."""
    r0, nl, rk, ws = _i64(), _i64(), _i32(), _i32()
    _chk(load().cwb_get_rows(ctx, C.byref(r0), C.byref(nl), C.byref(rk), C.byref(ws)), ctx)
    return r0.value, nl.value, rk.value, ws.value


class Pool:
    """RAII wrapper of a cwb_ctx."""

    def __init__(self, X, cfg: Config | None = None):
        self.ctx = cwb_init(X, cfg)
        self.n_star, self.d, self.K, self.n = cwb_get_dims(self.ctx)

    def status(self):
        cwb_status(self.ctx)

    def train(self, Y, nu=0.05, M=200, traces=True, out=None):
        return cwb_train(self.ctx, Y, nu, M, traces, out)

    def find_best(self, R):
        return cwb_find_best(self.ctx, R)

    def train_bernoulli(self, Y, nu=0.05, M=200, traces=True):
        return cwb_train_bernoulli(self.ctx, Y, nu, M, traces)

    def train_folds(self, Y, fold_of_row, F, fold_of_rep, nu=0.05, M=200):
        return cwb_train_folds(self.ctx, Y, fold_of_row, F, fold_of_rep, nu, M)

    def train_acwb(self, Y, nu=0.05, gamma=0.0034, M=200, traces=True):
        return cwb_train_acwb(self.ctx, Y, nu, gamma, M, traces)

    def train_hcwb(self, Y, val_mask, nu=0.05, gamma=0.037, pat0=5, M=200):
        return cwb_train_hcwb(self.ctx, Y, val_mask, nu, gamma, pat0, M)

    def predict(self, Xnew, offset, theta_agg):
        return cwb_predict(self.ctx, Xnew, offset, theta_agg)

    def set_path(self, p):
        cwb_set_path(self.ctx, p)

    def set_narrow(self, mode):
        cwb_set_narrow(self.ctx, mode)

    def lam(self):
        return cwb_get_lambda(self.ctx)

    def n_star_k(self):
        return cwb_get_n_star_k(self.ctx)

    def pool(self):
        return cwb_get_pool(self.ctx)

    def set_phase_timing(self, cycles4=None):
        cwb_set_phase_timing(self.ctx, cycles4)

    def launches(self):
        return cwb_launch_count(self.ctx)

    def set_h1_timing(self, on=True):
        cwb_set_h1_timing(self.ctx, on)

    def h1_time(self):
        return cwb_get_h1_time(self.ctx)

    def attach_learners(self, comm: Comm):
        _chk(load().cwb_attach_comm_learners(self.ctx, comm.h), self.ctx)
        self._comm = comm  # the communicator must outlive the context

    def attach(self, comm: Comm):
        cwb_attach_comm(self.ctx, comm)
        self._comm = comm  # the communicator must outlive the context
        self.n_star, self.d, self.K, self.n = cwb_get_dims(self.ctx)

    def rows(self):
        return cwb_get_rows(self.ctx)

    def close(self):
        if self.ctx:
            cwb_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
