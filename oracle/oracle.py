"""numpy/ctypes front end of the plain-C fp64 oracle (oracle/cwb_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py.  The product package
(paper_2110_03513_b200/) never imports this module and shares no code with it.

Every wrapper names the PAPER.md passage its C function follows (see
cwb_oracle.h).  Arrays are numpy float64 / int32, C-contiguous.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

MODE_DENSE, MODE_BINNED, MODE_UNBINNED = 0, 1, 2
_STATUS = {0: "OK", -1: "EINVAL", -2: "EDEGENERATE", -3: "ECALIB", -4: "ENONFINITE",
           -5: "EEMPTY", -8: "ENOMEM"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {_STATUS.get(code, code)}")
        self.code = code
        self.name = _STATUS.get(code, str(code))


def build() -> str:
    """Compile liboracle.so (plain gcc, -ffp-contract=off)."""
    src = os.path.join(_HERE, "cwb_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(src),
                                                 os.path.getmtime(os.path.join(_HERE, "cwb_oracle.h")))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None
_P = np.ctypeslib.ndpointer
_D = _P(dtype=np.float64, flags="C_CONTIGUOUS")
_I = _P(dtype=np.int32, flags="C_CONTIGUOUS")


class _Cfg(C.Structure):
    _fields_ = [("n_star_rule", C.c_int32), ("n_star_fixed", C.c_int32), ("degree", C.c_int32),
                ("n_knots", C.c_int32), ("df", C.c_double), ("df_kind", C.c_int32)]


class _Pool(C.Structure):
    _fields_ = [("K", C.c_int), ("n_star", C.c_int), ("d", C.c_int), ("mode", C.c_int),
                ("n", C.c_int64),
                ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double)),
                ("z", C.POINTER(C.c_double)), ("bnd", C.POINTER(C.c_double)),
                ("idx", C.POINTER(C.c_int32)), ("Zb", C.POINTER(C.c_double)),
                ("Zx", C.POINTER(C.c_double)), ("G", C.POINTER(C.c_double)),
                ("D", C.POINTER(C.c_double)), ("lam", C.POINTER(C.c_double)),
                ("L", C.POINTER(C.c_double)), ("degree", C.c_int), ("n_knots", C.c_int),
                ("nsk", C.POINTER(C.c_int32))]


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_n_star.argtypes = [C.c_int64, C.c_int, C.c_int]
        L.orc_build_bins.argtypes = [_D, C.c_int64, C.c_int, _D, _D, _I]
        L.orc_basis_dim.argtypes = [C.c_int, C.c_int]
        L.orc_bspline_basis.argtypes = [_D, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_int, _D]
        L.orc_penalty.argtypes = [C.c_int, _D]
        L.orc_penalty.restype = None
        L.orc_bin_mat_mat.argtypes = [_D, C.c_int, C.c_int, _I, C.c_void_p, C.c_int64, _D]
        L.orc_bin_mat_mat.restype = None
        L.orc_bin_mat_vec.argtypes = [_D, C.c_int, C.c_int, _I, C.c_void_p, _D, C.c_int64, _D]
        L.orc_bin_mat_vec.restype = None
        L.orc_dense_ztwz.argtypes = [_D, C.c_int, _I, C.c_void_p, C.c_int64, _D]
        L.orc_dense_ztwz.restype = None
        L.orc_dense_ztwr.argtypes = [_D, C.c_int, _I, C.c_void_p, _D, C.c_int64, _D]
        L.orc_dense_ztwr.restype = None
        L.orc_cholesky.argtypes = [_D, C.c_int, _D]
        L.orc_chol_solve.argtypes = [_D, C.c_int, _D, _D]
        L.orc_df.argtypes = [_D, _D, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.orc_df_to_lambda.argtypes = [_D, _D, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.orc_pool_new.argtypes = [_D, C.c_int64, C.c_int, C.POINTER(_Cfg), C.c_int,
                                   C.POINTER(C.POINTER(_Pool))]
        L.orc_pool_free.argtypes = [C.POINTER(_Pool)]
        L.orc_pool_free.restype = None
        L.orc_find_best.argtypes = [C.POINTER(_Pool), _D, C.POINTER(C.c_int32), _D,
                                    C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_double)]
        L.orc_train.argtypes = [C.POINTER(_Pool), _D, C.c_int, C.c_double, C.c_int, C.c_int,
                                _D, _D, _I, _D, _D, C.c_void_p, C.c_void_p]
        L.orc_train_loss.argtypes = [C.POINTER(_Pool), _D, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                     _D, _D, _I, _D, _D, C.c_void_p, C.c_void_p]
        L.orc_train_folds.argtypes = [C.POINTER(_Pool), _D, C.c_int, _P(dtype=np.uint8, flags="C_CONTIGUOUS"), C.c_int,
                                      _I, C.c_double, C.c_int, C.c_int, _D, _D, _I, _D, _D, _D, C.c_void_p,
                                      C.c_void_p]
        L.orc_train_follow.argtypes = [C.POINTER(_Pool), _D, C.c_int, C.c_double, C.c_int, C.c_int, _I, C.c_double,
                                       _D, _D, _I, _D, _D, C.c_void_p, C.c_void_p, _I]
        L.orc_train_acwb.argtypes = [C.c_void_p, _D, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int, _D, _D, _D,
                                     _I, _I, _D, _D, _D, _D, _D, _D, _D]
        L.orc_train_hcwb.argtypes = [C.c_void_p, _D, C.c_int, _P(dtype=np.uint8, flags="C_CONTIGUOUS"), C.c_double,
                                     C.c_double, C.c_int, C.c_int, C.c_int, _D, _D, _I, _I, _D, _D, _D, _I, _D, _D, _D]
        L.orc_predict.argtypes = [C.POINTER(_Pool), _D, C.c_int64, _D, _D, C.c_int, _D]
        _lib = L
    return _lib


def _chk(code: int, where: str) -> None:
    if code != 0:
        raise OracleError(code, where)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _wptr(w):
    if w is None:
        return None, None
    w = _f64(w)
    return w, w.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- primitives

def n_star(n: int, rule: int = 0, fixed: int = 0) -> int:
    """P:L859 / P:L445 bin-count rule."""
    v = lib().orc_n_star(n, rule, fixed)
    if v < 0:
        raise OracleError(v, "n_star")
    return v


def build_bins(x, ns: int):
    """design points z, boundaries, 0-based index vector."""
    x = _f64(x)
    z = np.empty(ns)
    bnd = np.empty(max(ns - 1, 1))
    idx = np.empty(len(x), dtype=np.int32)
    _chk(lib().orc_build_bins(x, len(x), ns, z, bnd, idx), "build_bins")
    return z, bnd[: ns - 1], idx


def basis_dim(degree: int = 3, n_knots: int = 20) -> int:
    return lib().orc_basis_dim(degree, n_knots)


def bspline_basis(x, lo: float, hi: float, degree: int = 3, n_knots: int = 20) -> np.ndarray:
    """P:L822 Cox-de Boor B-spline basis on extended equidistant knots."""
    x = _f64(x)
    d = basis_dim(degree, n_knots)
    out = np.empty((len(x), d))
    _chk(lib().orc_bspline_basis(x, len(x), lo, hi, degree, n_knots, out), "bspline_basis")
    return out


def penalty(d: int) -> np.ndarray:
    """Supp. P:L312 second-order difference penalty."""
    D = np.empty((d, d))
    lib().orc_penalty(d, D)
    return D


def bin_mat_mat(Zb, idx, w=None) -> np.ndarray:
    """Algorithm binMatMat."""
    Zb = _f64(Zb)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    w, wp = _wptr(w)
    out = np.empty((Zb.shape[1], Zb.shape[1]))
    lib().orc_bin_mat_mat(Zb, Zb.shape[0], Zb.shape[1], idx, wp, len(idx), out)
    return out


def bin_mat_vec(Zb, idx, r, w=None) -> np.ndarray:
    """Algorithm binMatVec."""
    Zb = _f64(Zb)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    r = _f64(r)
    w, wp = _wptr(w)
    out = np.empty(Zb.shape[1])
    lib().orc_bin_mat_vec(Zb, Zb.shape[0], Zb.shape[1], idx, wp, r, len(idx), out)
    return out


def dense_ztwz(Zb, idx, w=None) -> np.ndarray:
    Zb = _f64(Zb)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    w, wp = _wptr(w)
    out = np.empty((Zb.shape[1], Zb.shape[1]))
    lib().orc_dense_ztwz(Zb, Zb.shape[1], idx, wp, len(idx), out)
    return out


def dense_ztwr(Zb, idx, r, w=None) -> np.ndarray:
    Zb = _f64(Zb)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    r = _f64(r)
    w, wp = _wptr(w)
    out = np.empty(Zb.shape[1])
    lib().orc_dense_ztwr(Zb, Zb.shape[1], idx, wp, r, len(idx), out)
    return out


def cholesky(A) -> np.ndarray:
    A = _f64(A)
    L = np.empty_like(A)
    _chk(lib().orc_cholesky(A, A.shape[0], L), "cholesky")
    return L


def chol_solve(A, b) -> np.ndarray:
    A, b = _f64(A), _f64(b)
    x = np.empty_like(b)
    _chk(lib().orc_chol_solve(A, A.shape[0], b, x), "chol_solve")
    return x


def df(G, D, lam: float, kind: int = 1) -> float:
    """Supp. P:L314-318 df1 = tr H, df2 = tr(2H - H^2)."""
    G, D = _f64(G), _f64(D)
    out = C.c_double()
    _chk(lib().orc_df(G, D, G.shape[0], lam, kind, C.byref(out)), "df")
    return out.value


def df_to_lambda(G, D, target: float, kind: int = 1) -> float:
    G, D = _f64(G), _f64(D)
    out = C.c_double()
    _chk(lib().orc_df_to_lambda(G, D, G.shape[0], target, kind, C.byref(out)), "df_to_lambda")
    return out.value


# ---------------------------------------------------------------- pool/train

@dataclass
class Config:
    n_star_rule: int = 0      # 0 ceil(sqrt n), 1 ceil(n^(1/4)), 2 fixed
    n_star_fixed: int = 0
    degree: int = 3
    n_knots: int = 20
    df: float = 5.0
    df_kind: int = 1

    def _c(self) -> _Cfg:
        return _Cfg(self.n_star_rule, self.n_star_fixed, self.degree, self.n_knots, self.df, self.df_kind)


@dataclass
class TrainResult:
    offset: np.ndarray      # B
    theta_agg: np.ndarray   # B x K x d
    k_trace: np.ndarray     # M x B
    sse_trace: np.ndarray   # M x B
    risk_trace: np.ndarray  # M x B
    gap_trace: np.ndarray   # M x B  (SSE second best - SSE best)
    f: np.ndarray           # B x n  final fit


@dataclass
class AcwbResult:
    offset: np.ndarray        # B
    theta_f: np.ndarray       # B x K x d  primary model parameters
    theta_h: np.ndarray       # B x K x d  momentum model parameters
    k_trace: np.ndarray       # M x B
    kcor_trace: np.ndarray    # M x B
    sse_trace: np.ndarray     # M x B
    sse_cor_trace: np.ndarray  # M x B
    risk_trace: np.ndarray    # M x B  risk of f after iteration m
    gap_trace: np.ndarray     # M x B
    gap_cor_trace: np.ndarray  # M x B
    f: np.ndarray             # B x n
    h: np.ndarray             # B x n


@dataclass
class HcwbResult:
    offset: np.ndarray          # B
    theta_f: np.ndarray         # B x K x d
    k_trace: np.ndarray         # M x B
    kcor_trace: np.ndarray      # M x B (-1 after the switch)
    sse_trace: np.ndarray       # M x B
    risk_trace: np.ndarray      # M x B  risk of f on all rows
    val_risk_trace: np.ndarray  # M x B  risk of f on the validation rows
    switch_iter: np.ndarray     # B
    gap_trace: np.ndarray       # M x B
    gap_cor_trace: np.ndarray   # M x B
    f: np.ndarray               # B x n


class Pool:
    """K binned P-spline base learners on X (K x n)."""

    def __init__(self, X, cfg: Config | None = None, mode: int = MODE_BINNED):
        X = _f64(X)
        self.cfg = cfg or Config()
        K, n = X.shape
        p = C.POINTER(_Pool)()
        _chk(lib().orc_pool_new(X, n, K, C.byref(self.cfg._c()), mode, C.byref(p)), "pool_new")
        self._p = p
        s = p.contents
        self.K, self.n, self.n_star, self.d, self.mode = s.K, s.n, s.n_star, s.d, s.mode
        K, ns, d = self.K, self.n_star, self.d

        def arr(ptr, shape, dt=np.float64):
            return np.ctypeslib.as_array(ptr, shape=shape).astype(dt, copy=True)

        self.lo = arr(s.lo, (K,))
        self.hi = arr(s.hi, (K,))
        self.z = arr(s.z, (K, ns))
        self.bnd = arr(s.bnd, (K, ns - 1))
        self.idx = arr(s.idx, (K, self.n), np.int32)
        self.Zb = arr(s.Zb, (K, ns, d))
        self.G = arr(s.G, (K, d, d))
        self.D = arr(s.D, (d, d))
        self.lam = arr(s.lam, (K,))
        self.nsk = arr(s.nsk, (K,), np.int32)  # effective bins per learner (S:L143 clamp, reading N1)

    def __del__(self):
        p = getattr(self, "_p", None)
        if p is not None and _lib is not None:
            _lib.orc_pool_free(p)
            self._p = None

    def find_best(self, r):
        """findBestBaselearner, P:L927 / Alg. 1 supp. lines 5-9."""
        r = _f64(r)
        k = C.c_int32()
        theta = np.empty(self.d)
        sse = C.c_double()
        gap = C.c_double()
        sse_all = np.empty(self.K)
        _chk(lib().orc_find_best(self._p, r, C.byref(k), theta, C.byref(sse),
                                 sse_all.ctypes.data_as(C.c_void_p), C.byref(gap)), "find_best")
        return int(k.value), theta, sse.value, sse_all, gap.value

    def train(self, Y, nu: float = 0.05, M: int = 200, threads: int = 1) -> TrainResult:
        """Alg. 1 supp. for B target vectors Y (B x n)."""
        Y = _f64(np.atleast_2d(Y))
        B = Y.shape[0]
        K, d = self.K, self.d
        off = np.empty(B)
        agg = np.empty((B, K, d))
        kt = np.empty((M, B), dtype=np.int32)
        st = np.empty((M, B))
        rt = np.empty((M, B))
        gt = np.empty((M, B))
        f = np.empty((B, self.n))
        _chk(lib().orc_train(self._p, Y, B, nu, M, threads, off, agg, kt, st, rt,
                             gt.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p)), "train")
        return TrainResult(off, agg, kt, st, rt, gt, f)

    def train_follow(self, Y, follow, tie_rtol: float = 1e-10, nu: float = 0.05, M: int = 200, threads: int = 1):
        """Alg. 1 supp. in tie-following mode: at a near-tie (SSE within tie_rtol of the minimum) the
        learner follow[m][b] is taken.  Returns (TrainResult, followed[B])."""
        Y = _f64(np.atleast_2d(Y))
        B = Y.shape[0]
        K, d = self.K, self.d
        off = np.empty(B)
        agg = np.empty((B, K, d))
        kt = np.empty((M, B), dtype=np.int32)
        st = np.empty((M, B))
        rt = np.empty((M, B))
        gt = np.empty((M, B))
        f = np.empty((B, self.n))
        fol = np.zeros(B, dtype=np.int32)
        _chk(lib().orc_train_follow(self._p, Y, B, nu, M, threads, np.ascontiguousarray(follow, dtype=np.int32),
                                    tie_rtol, off, agg, kt, st, rt, gt.ctypes.data_as(C.c_void_p),
                                    f.ctypes.data_as(C.c_void_p), fol), "train_follow")
        return TrainResult(off, agg, kt, st, rt, gt, f), fol

    def train_bernoulli(self, Y, nu: float = 0.05, M: int = 200, threads: int = 1) -> TrainResult:
        """Alg. 1 supp. with the Bernoulli loss, y in {0, 1}, for B
        target vectors Y (B x n); risk_trace = mean log-loss after iteration m."""
        Y = _f64(np.atleast_2d(Y))
        B = Y.shape[0]
        K, d = self.K, self.d
        off = np.empty(B)
        agg = np.empty((B, K, d))
        kt = np.empty((M, B), dtype=np.int32)
        st = np.empty((M, B))
        rt = np.empty((M, B))
        gt = np.empty((M, B))
        f = np.empty((B, self.n))
        _chk(lib().orc_train_loss(self._p, Y, B, 1, nu, M, threads, off, agg, kt, st, rt,
                                  gt.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p)), "train_bernoulli")
        return TrainResult(off, agg, kt, st, rt, gt, f)

    def train_folds(self, Y, fold_of_row, F: int, fold_of_rep, nu: float = 0.05, M: int = 200, threads: int = 1):
        """CWB with per-replication 0/1 observation weights (CV folds): replication b
        fits on the rows with fold_of_row != fold_of_rep[b]; returns (TrainResult, val_risk_trace)."""
        Y = _f64(np.atleast_2d(Y))
        B = Y.shape[0]
        K, d = self.K, self.d
        off = np.empty(B)
        agg = np.empty((B, K, d))
        kt = np.empty((M, B), dtype=np.int32)
        st = np.empty((M, B))
        rt = np.empty((M, B))
        vt = np.empty((M, B))
        gt = np.empty((M, B))
        f = np.empty((B, self.n))
        _chk(lib().orc_train_folds(self._p, Y, B, np.ascontiguousarray(fold_of_row, dtype=np.uint8), F,
                                   np.ascontiguousarray(fold_of_rep, dtype=np.int32), nu, M, threads, off, agg, kt,
                                   st, rt, vt, gt.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p)),
             "train_folds")
        return TrainResult(off, agg, kt, st, rt, gt, f), vt

    def train_acwb(self, Y, nu: float = 0.05, gamma: float = 0.0034, M: int = 200,
                   threads: int = 1) -> AcwbResult:
        """Accelerated CWB, Algorithm 2, for B target vectors Y (B x n)."""
        Y = _f64(np.atleast_2d(Y))
        B = Y.shape[0]
        K, d, n = self.K, self.d, self.n
        off = np.empty(B)
        tf = np.empty((B, K, d))
        th = np.empty((B, K, d))
        kt = np.empty((M, B), dtype=np.int32)
        kc = np.empty((M, B), dtype=np.int32)
        st, sc, rt, gt, gc = (np.empty((M, B)) for _ in range(5))
        f = np.empty((B, n))
        h = np.empty((B, n))
        _chk(lib().orc_train_acwb(C.cast(self._p, C.c_void_p), Y, B, nu, gamma, M, threads, off, tf, th, kt, kc,
                                  st, sc, rt, gt, gc, f, h), "train_acwb")
        return AcwbResult(off, tf, th, kt, kc, st, sc, rt, gt, gc, f, h)

    def train_hcwb(self, Y, val_mask, nu: float = 0.05, gamma: float = 0.037, pat0: int = 5, M: int = 200,
                   threads: int = 1) -> HcwbResult:
        """Hybrid CWB, Algorithm 3; val_mask[n] = 1 for validation rows."""
        Y = _f64(np.atleast_2d(Y))
        B = Y.shape[0]
        K, d, n = self.K, self.d, self.n
        vm = np.ascontiguousarray(val_mask, dtype=np.uint8)
        off = np.empty(B)
        tf = np.empty((B, K, d))
        kt = np.empty((M, B), dtype=np.int32)
        kc = np.empty((M, B), dtype=np.int32)
        st, rt, vt, gt, gc = (np.empty((M, B)) for _ in range(5))
        sw = np.empty(B, dtype=np.int32)
        f = np.empty((B, n))
        _chk(lib().orc_train_hcwb(C.cast(self._p, C.c_void_p), Y, B, vm, nu, gamma, pat0, M, threads, off, tf, kt, kc,
                                  st, rt, vt, sw, gt, gc, f), "train_hcwb")
        return HcwbResult(off, tf, kt, kc, st, rt, vt, sw, gt, gc, f)

    def predict(self, Xnew, offset, theta_agg) -> np.ndarray:
        Xnew = _f64(Xnew)
        offset = _f64(np.atleast_1d(offset))
        theta_agg = _f64(theta_agg).reshape(len(offset), self.K, self.d)
        out = np.empty((len(offset), Xnew.shape[1]))
        _chk(lib().orc_predict(self._p, Xnew, Xnew.shape[1], offset, theta_agg, len(offset), out),
             "predict")
        return out
