"""ctypes wrapper for oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.

The oracle is a plain, literal CPU FP64 implementation of one refinement sweep
(Alg. 4, with Alg. 2/3 for the WY factors).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu-baseline / `--impl reference` legs
may import this package.  It shares no code with paper_2602_23778_b200 and
never imports it.

All arrays are numpy float64 (int32 for CSR indices), row-major n x k.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

# status values (oracle.c enum)
OK, MAXITER, DIVERGED, E_INVALID, E_NEAR_ZERO_RQ, E_ZERO_PIVOT, E_NOMEM = 0, 1, 2, -1, -2, -3, -6

CFLAGS = ["-O2", "-ffp-contract=off", "-mavx2", "-mfma", "-fopenmp", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-ffp-contract=off: every fma in the oracle is explicit)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class Stats(C.Structure):
    _fields_ = [("rel_resid", C.c_double), ("corr_norm", C.c_double), ("min_gap", C.c_double),
                ("delta_hits", C.c_int32), ("flipped", C.c_int32), ("gram_dev", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i64, i32, d = C.c_int64, C.c_int32, C.c_double
        L.oracle_norm_inf_dense.argtypes = [i64, P, i64, d]; L.oracle_norm_inf_dense.restype = d
        L.oracle_norm_inf_csr.argtypes = [i64, P, P, P, d]; L.oracle_norm_inf_csr.restype = d
        L.oracle_apply_dense.argtypes = [i64, i32, P, i64, d, P, P]
        L.oracle_apply_csr.argtypes = [i64, i32, P, P, P, d, P, P]
        L.oracle_modified_lu.argtypes = [i64, i32, P, P]
        L.oracle_compact_wy_lu.argtypes = [i64, i32, P, P, P, P, P]
        L.oracle_compact_wy.argtypes = [i64, i32, P, P, P]
        L.oracle_apply_h.argtypes = [i64, i32, P, P, i32, P, P, C.c_int]
        L.oracle_sweep_dense.argtypes = [i64, i32, P, i64, d, P, d, i32, i32, C.POINTER(Stats), P]
        L.oracle_sweep_csr.argtypes = [i64, i32, P, P, P, d, P, d, i32, i32, C.POINTER(Stats), P]
        L.oracle_run_dense.argtypes = [i64, i32, P, i64, d, P, i32, d, d, i32, i32, d, C.POINTER(i32), P]
        L.oracle_run_csr.argtypes = [i64, i32, P, P, P, d, P, i32, d, d, i32, i32, d, C.POINTER(i32), P]
        L.oracle_rr_dense.argtypes = [i64, i32, P, i64, d, P, P]
        L.oracle_rr_csr.argtypes = [i64, i32, P, P, P, d, P, P]
        L.oracle_jacobi_eig.argtypes = [i32, P, P, P]
        L.oracle_sweep_tz_dense.argtypes = [i64, i32, P, i64, d, P, d, C.POINTER(Stats), P]
        L.oracle_sweep_tz_csr.argtypes = [i64, i32, P, P, P, d, P, d, C.POINTER(Stats), P]
        L.oracle_sweep_ex.argtypes = [C.c_int, i64, i32, P, i64, P, P, P, d, i32, P, d, i32, i32, i32, C.POINTER(Stats), P]
        L.oracle_run_ex.argtypes = [C.c_int, i64, i32, P, i64, P, P, P, d, i32, P, i32, d, d, i32, i32,
                                    C.POINTER(i32), P]
        L.oracle_apply_ex.argtypes = [C.c_int, i64, i32, P, i64, P, P, P, d, i32, P, P]
        L.oracle_norm_ex.argtypes = [C.c_int, i64, P, i64, P, P, P, d, i32]
        L.oracle_norm_ex.restype = d
        L.oracle_reorthogonalize.argtypes = [i64, i32, P, P]
        L.oracle_num_threads.restype = C.c_int
        for f in ("oracle_apply_dense", "oracle_apply_csr", "oracle_modified_lu", "oracle_compact_wy_lu",
                  "oracle_compact_wy", "oracle_apply_h", "oracle_sweep_dense", "oracle_sweep_csr",
                  "oracle_run_dense", "oracle_run_csr"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Operator:
    """A (dense n x n, or CSR with both triangles) and the Sec. 5.1 shift;
    square=True: the operator A^2 - shift I of Sec. 5.2, applied as A (A X)."""

    def __init__(self, A=None, row_ptr=None, col_idx=None, val=None, shift: float = 0.0, square: bool = False):
        self.shift = float(shift)
        self.square = bool(square)
        if A is not None:
            self.is_csr = False
            self.A = _f64(A)
            self.n = self.A.shape[0]
        else:
            self.is_csr = True
            self.rp, self.ci, self.v = _i32(row_ptr), _i32(col_idx), _f64(val)
            self.n = self.rp.size - 1

    def norm_inf(self) -> float:
        L = lib()
        if self.square:
            a = _ex_args(self)
            return L.oracle_norm_ex(*a)
        if self.is_csr:
            return L.oracle_norm_inf_csr(self.n, _p(self.rp), _p(self.ci), _p(self.v), self.shift)
        return L.oracle_norm_inf_dense(self.n, _p(self.A), self.n, self.shift)

    def apply(self, X) -> np.ndarray:
        """W = A X - shift X (Alg. 4 line 1), fma chain in ascending column order."""
        X = _f64(X)
        k = X.shape[1]
        W = np.empty_like(X)
        L = lib()
        if self.square:
            a = _ex_args(self)
            L.oracle_apply_ex(*a[:2], k, *a[2:], _p(X), _p(W))
            return W
        if self.is_csr:
            L.oracle_apply_csr(self.n, k, _p(self.rp), _p(self.ci), _p(self.v), self.shift, _p(X), _p(W))
        else:
            L.oracle_apply_dense(self.n, k, _p(self.A), self.n, self.shift, _p(X), _p(W))
        return W


def modified_lu(Q):
    """Alg. 2.  Returns (Y unit-lower n x k, U k x k, sigma k, status)."""
    Q = _f64(Q).copy()
    n, k = Q.shape
    sig = np.zeros(k)
    st = lib().oracle_modified_lu(n, k, _p(Q), _p(sig))
    Y = np.tril(Q, -1)
    Y[np.arange(k), np.arange(k)] = 1.0
    U = np.triu(Q[:k])
    return Y, U, sig, st


def compact_wy_lu(Q):
    """Alg. 3.  Returns (Y, T, sigma, U, status)."""
    Q = _f64(Q)
    n, k = Q.shape
    Y, T, sig, U = np.zeros((n, k)), np.zeros((k, k)), np.zeros(k), np.zeros((k, k))
    st = lib().oracle_compact_wy_lu(n, k, _p(Q), _p(Y), _p(T), _p(sig), _p(U))
    return Y, T, sig, U, st


def compact_wy(Q):
    """Alg. 1.  Returns (Y, T, status)."""
    Q = _f64(Q)
    n, k = Q.shape
    Y, T = np.zeros((n, k)), np.zeros((k, k))
    st = lib().oracle_compact_wy(n, k, _p(Q), _p(Y), _p(T))
    return Y, T, st


def apply_h(Y, T, B, transpose=False):
    """H B = B - Y(T(Y^T B)) or H^T B."""
    Y, T, B = _f64(Y), _f64(T), _f64(B)
    n, k = Y.shape
    m = B.shape[1]
    out = np.empty_like(B)
    lib().oracle_apply_h(n, k, _p(Y), _p(T), m, _p(B), _p(out), int(transpose))
    return out


DEBUG_KEYS = ("W", "Y", "T", "sigma", "dtilde", "alpha", "V", "E", "Xtilde", "U")


def _debug_buffers(n, k, debug):
    """Host arrays for the sweep's intermediate dumps (oracle.c DBG_*) and the pointer table."""
    if not debug:
        return {}, None
    shapes = {"W": (n, k), "Y": (n, k), "T": (k, k), "sigma": (k,), "dtilde": (k,), "alpha": (k,),
              "V": (n, k), "E": (n, k), "Xtilde": (n, k), "U": (k, k)}
    dbg = {key: np.zeros(shapes[key]) for key in DEBUG_KEYS}
    arr = (C.c_void_p * len(DEBUG_KEYS))(*[dbg[key].ctypes.data for key in DEBUG_KEYS])
    dbg["_keep"] = arr
    return dbg, C.cast(arr, C.c_void_p)


@dataclass
class SweepResult:
    X: np.ndarray
    status: int
    stats: Stats
    debug: dict


def _ex_args(op):
    if op.is_csr:
        return (1, op.n, None, 0, _p(op.rp), _p(op.ci), _p(op.v), op.shift, int(op.square))
    return (0, op.n, _p(op.A), op.n, None, None, None, op.shift, int(op.square))


def sweep(op: Operator, X, delta_c=10.0, beta_zero=False, normalize=True, debug=False, kjudge=0,
          want_gram=False) -> SweepResult:
    """One sweep of Alg. 4 on a copy of X.  kjudge > 0: corr_norm over the leading
    kjudge columns (K > k refinement); want_gram: stats.gram_dev (else -1)."""
    if op.square or kjudge or want_gram:
        assert normalize and not debug
        X = _f64(X).copy()
        n, k = X.shape
        st = Stats()
        a = _ex_args(op)
        s = lib().oracle_sweep_ex(*a[:2], k, *a[2:], _p(X), delta_c, int(beta_zero), int(kjudge), int(want_gram),
                                  C.byref(st), None)
        return SweepResult(X, s, st, {})
    X = _f64(X).copy()
    n, k = X.shape
    st = Stats()
    dbg, dptr = _debug_buffers(n, k, debug)
    L = lib()
    if op.is_csr:
        s = L.oracle_sweep_csr(n, k, _p(op.rp), _p(op.ci), _p(op.v), op.shift, _p(X), delta_c, int(beta_zero),
                               int(normalize), C.byref(st), dptr)
    else:
        s = L.oracle_sweep_dense(n, k, _p(op.A), n, op.shift, _p(X), delta_c, int(beta_zero), int(normalize),
                                 C.byref(st), dptr)
    return SweepResult(X, s, st, dbg)


def run(op: Operator, X, iters: int, tol: float, delta_c=10.0, beta_zero=False, guard_window=3,
        guard_factor=10.0, kjudge=0):
    """Iterate sweeps until ||E_L||_F <= tol, iters, or divergence.
    Returns (X, status, iters_done, history[iters_done, 2] = (rel_resid, corr_norm))."""
    X = _f64(X).copy()
    n, k = X.shape
    hist = np.zeros((max(iters, 1), 2))
    done = C.c_int32(0)
    L = lib()
    if op.square or kjudge:     # (no divergence guard on this entry point)
        a = _ex_args(op)
        s = L.oracle_run_ex(*a[:2], k, *a[2:], _p(X), iters, tol, delta_c, int(beta_zero), int(kjudge),
                            C.byref(done), _p(hist))
        return X, s, done.value, hist[:done.value]
    if op.is_csr:
        s = L.oracle_run_csr(n, k, _p(op.rp), _p(op.ci), _p(op.v), op.shift, _p(X), iters, tol, delta_c,
                             int(beta_zero), guard_window, guard_factor, C.byref(done), _p(hist))
    else:
        s = L.oracle_run_dense(n, k, _p(op.A), n, op.shift, _p(X), iters, tol, delta_c, int(beta_zero),
                               guard_window, guard_factor, C.byref(done), _p(hist))
    return X, s, done.value, hist[:done.value]


def rayleigh_ritz(op: Operator, X):
    """Rayleigh-Ritz preprocessing (Sec. 3.4): returns (status, Z, ritz) with
    Z = X S, (X^T A X) S = (X^T X) S diag(ritz); ritz descending (readings RR1-RR3 in oracle.c)."""
    Z = np.array(X, dtype=np.float64, order="C", copy=True)
    n, k = Z.shape
    ritz = np.zeros(k)
    if not op.is_csr:
        s = lib().oracle_rr_dense(n, k, _p(op.A), op.n, op.shift, _p(Z), _p(ritz))
    else:
        s = lib().oracle_rr_csr(n, k, _p(op.rp), _p(op.ci), _p(op.v), op.shift, _p(Z), _p(ritz))
    return s, Z, ritz


def sweep_rr(op: Operator, X, delta_c=10.0, debug=False):
    """Rayleigh-Ritz (Sec. 3.4) followed by one sweep with the top block of E_L zero and beta = 0
    (PAPER.md:460, 921-926): one iteration of the preprocessed refinement.  Returns
    (SweepResult, ritz); the result's status is the RR status if RR fails.  debug: the top-zero
    sweep's intermediates (as in sweep(); its input is the RR output Z, kept in debug["Z"])."""
    s, Z, ritz = rayleigh_ritz(op, X)
    st = Stats()
    if s != OK:
        return SweepResult(Z, s, st, {}), ritz
    n, k = Z.shape
    dbg, dptr = _debug_buffers(n, k, debug)
    if debug:
        dbg["Z"] = Z.copy()
    L = lib()
    if op.is_csr:
        s = L.oracle_sweep_tz_csr(n, k, _p(op.rp), _p(op.ci), _p(op.v), op.shift, _p(Z), delta_c, C.byref(st), dptr)
    else:
        s = L.oracle_sweep_tz_dense(n, k, _p(op.A), n, op.shift, _p(Z), delta_c, C.byref(st), dptr)
    return SweepResult(Z, s, st, dbg), ritz


def reorthogonalize(X):
    """Cholesky-QR reorthogonalisation X <- X L^{-T} (NEXT-4).  Returns (status, Z, gram_dev)."""
    Z = np.array(X, dtype=np.float64, order="C", copy=True)
    n, k = Z.shape
    gd = C.c_double(0.0)
    s = lib().oracle_reorthogonalize(n, k, _p(Z), C.byref(gd))
    return s, Z, gd.value


def run_policy(op: Operator, X, iters: int, tol: float, resid_tol: float = 0.0, reorth_tol: float = 0.0,
               rr_fallback: bool = False, delta_c=10.0, beta_zero=False, guard_window=3, guard_factor=10.0):
    """refine_run with the NEXT-4 policies (the loop is plain Python over the oracle's C sweeps):
      * stop when ||E_L||_F <= tol or, resid_tol > 0, when the relative residual
        ||A X - X D||_F / ||A|| <= resid_tol;
      * reorth_tol > 0: when a sweep's input has max|X^T X - I| > reorth_tol, reorthogonalise its
        output (Cholesky QR);
      * the divergence guard (||E_L||_F grows >= guard_factor within guard_window sweeps,
        PAPER.md:1155); rr_fallback: instead of stopping, continue with Rayleigh-Ritz iterations
        (Sec. 3.4, the paper's "terminate and switch to preprocessing").
    Returns (X, status, sweeps, history[(rel_resid, corr_norm, mode)]) with mode 0 = plain, 1 = RR."""
    X = _f64(X).copy()
    hist = []
    mode = 0
    cs = []
    for t in range(iters):
        if mode == 0:
            res = sweep(op, X, delta_c=delta_c, beta_zero=beta_zero, want_gram=reorth_tol > 0)
        else:
            res, _ = sweep_rr(op, X, delta_c=delta_c)
        if res.status != OK:
            return res.X, res.status, t + 1, np.array(hist)
        st = res.stats
        hist.append((st.rel_resid, st.corr_norm, mode))
        if not np.isfinite(st.corr_norm):
            return res.X, DIVERGED, t + 1, np.array(hist)
        X = res.X
        if st.corr_norm <= tol or (resid_tol > 0 and st.rel_resid <= resid_tol):
            return X, OK, t + 1, np.array(hist)
        cs.append(st.corr_norm)
        if mode == 0 and guard_window > 0 and len(cs) > guard_window and cs[-1] >= guard_factor * cs[-1 - guard_window]:
            if not rr_fallback:
                return X, DIVERGED, t + 1, np.array(hist)
            mode = 1
            continue
        if mode == 0 and reorth_tol > 0 and st.gram_dev > reorth_tol:
            s, X, _ = reorthogonalize(X)
            if s != OK:
                return X, s, t + 1, np.array(hist)
    return X, MAXITER, iters, np.array(hist)


def jacobi_eig(Cm):
    """k x k symmetric eigen-decomposition by cyclic Jacobi (oracle.c jacobi_eig): (Q, d), unsorted."""
    Cw = np.array(Cm, dtype=np.float64, order="C", copy=True)
    k = Cw.shape[0]
    Q, dv = np.zeros((k, k)), np.zeros(k)
    lib().oracle_jacobi_eig(k, _p(Cw), _p(Q), _p(dv))
    return Q, dv


def num_threads() -> int:
    return lib().oracle_num_threads()
