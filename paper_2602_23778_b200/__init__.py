"""paper_2602_23778_b200 -- B200-native refinement sweep for a subset of eigenvectors
(arXiv 2602.23778, Algorithm 4).

Thin ctypes binding of the C ABI in include/refine.h: argument marshalling only.
Every step of the sweep runs in the CUDA kernels of csrc/ (librefine.so, built for
sm_100a by `python -m paper_2602_23778_b200.build` or __graft_entry__.build()).
There is no CPU fallback: if the library is missing or no CUDA device is present,
calls raise.

PyTorch supplies device memory (tensor data pointers) and streams only.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librefine.so")

# refine_status (include/refine.h)
REFINE_OK, REFINE_MAXITER, REFINE_DIVERGED = 0, 1, 2
REFINE_E_INVALID, REFINE_E_NEAR_ZERO_RQ, REFINE_E_ZERO_PIVOT = -1, -2, -3
REFINE_E_CUDA, REFINE_E_NCCL, REFINE_E_NOMEM, REFINE_E_UNSUPPORTED = -4, -5, -6, -7

# refine_debug_get selectors
DBG_W, DBG_SIGMA, DBG_U, DBG_L, DBG_T, DBG_D, DBG_ALPHA, DBG_E11, DBG_Y, DBG_STATS = range(10)
DBG_SPMM = 11   # S1 kernel geometry: [stencil on, R, L, nq, grid, nx, ny, nz, gather R]


class refine_comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p)]


class refine_opts(C.Structure):
    _fields_ = [("delta_c", C.c_double), ("beta_zero", C.c_int32), ("normalize", C.c_int32),
                ("guard_window", C.c_int32), ("guard_factor", C.c_double), ("square", C.c_int32),
                ("kjudge", C.c_int32), ("resid_tol", C.c_double), ("reorth_tol", C.c_double),
                ("rr_fallback", C.c_int32), ("mixed", C.c_int32), ("emul", C.c_int32)]


class refine_sweep_stats(C.Structure):
    _fields_ = [("rel_resid", C.c_double), ("corr_norm", C.c_double), ("min_gap", C.c_double),
                ("delta_hits", C.c_int32), ("flipped", C.c_int32), ("gram_dev", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class RefineError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {refine_status_string(status)} ({status})")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Load librefine.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                              "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        P, i64, i32, d = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        L.refine_init_dense.argtypes = [C.POINTER(P), i64, i32, P, i64, i64, i64, d, C.POINTER(refine_comm),
                                        C.POINTER(refine_opts), P]
        L.refine_init_csr.argtypes = [C.POINTER(P), i64, i32, P, P, P, i64, i64, d, C.POINTER(refine_comm),
                                      C.POINTER(refine_opts), P]
        L.refine_sweep.argtypes = [P, P, C.POINTER(refine_sweep_stats)]
        L.refine_sweep_host.argtypes = [P, P, P, C.POINTER(refine_sweep_stats)]
        L.refine_run.argtypes = [P, P, i32, d, C.POINTER(i32), C.POINTER(refine_sweep_stats)]
        L.refine_get_status.argtypes = [P]
        L.refine_set_graph.argtypes = [P, i32]
        L.refine_kernels_per_sweep.argtypes = [P]
        L.refine_kernels_per_sweep.restype = i32
        L.refine_destroy.argtypes = [P]
        L.refine_destroy.restype = None
        L.refine_status_string.argtypes = [C.c_int]
        L.refine_status_string.restype = C.c_char_p
        L.refine_nccl_id.argtypes = [P]
        L.refine_debug_get.argtypes = [P, i32, P]
        L.refine_profile_begin.argtypes = [P, i32]
        L.refine_profile_end.argtypes = [P, C.POINTER(C.c_double), C.POINTER(i32), C.POINTER(i32)]
        L.refine_kernel_name.argtypes = [P, i32]
        L.refine_kernel_name.restype = C.c_char_p
        L.refine_halo_plan.argtypes = [i32, i32, P, P, P, P, P, C.POINTER(i32), P, C.POINTER(i32), C.POINTER(i64), i32]
        L.refine_halo_plan.restype = i32
        L.refine_rayleigh_ritz.argtypes = [P, P, P]
        L.refine_sweep_rr.argtypes = [P, P, C.POINTER(refine_sweep_stats), P]
        L.refine_reorthogonalize.argtypes = [P, P, P]
        for f in ("refine_init_dense", "refine_init_csr", "refine_sweep", "refine_sweep_host", "refine_run",
                  "refine_get_status", "refine_set_graph", "refine_nccl_id", "refine_debug_get",
                  "refine_profile_begin", "refine_profile_end", "refine_rayleigh_ritz", "refine_sweep_rr",
                  "refine_reorthogonalize"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def refine_status_string(s: int) -> str:
    return lib().refine_status_string(int(s)).decode()


def _ptr(t) -> int:
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _check_dev(t, dtype, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous CUDA tensor of dtype {dtype}")


def _opts(delta_c=10.0, beta_zero=False, normalize=True, guard_window=3, guard_factor=10.0, square=False, kjudge=0,
          resid_tol=0.0, reorth_tol=0.0, rr_fallback=False, mixed=False, emul=False):
    return refine_opts(float(delta_c), int(bool(beta_zero)), int(bool(normalize)), int(guard_window),
                       float(guard_factor), int(bool(square)), int(kjudge), float(resid_tol), float(reorth_tol),
                       int(bool(rr_fallback)), int(mixed), int(bool(emul)))


@dataclass
class _Keep:
    tensors: tuple


class Refiner:
    """Context of the sweep (refine_ctx).  A and its CSR arrays are borrowed: the
    Refiner keeps Python references to the tensors so they outlive the context."""

    def __init__(self, handle: int, n: int, k: int, n_loc: int, keep: tuple, stream):
        self._h = C.c_void_p(handle)
        self.n, self.k, self.n_loc = n, k, n_loc
        self._keep = keep
        self._stream = stream

    # -- construction -------------------------------------------------------------
    @classmethod
    def dense(cls, A, k: int, shift: float = 0.0, row_begin: int = 0, row_end: int | None = None,
              n: int | None = None, stream=None, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
              **opts) -> "Refiner":
        """refine_init_dense: A is (row_end-row_begin) x n float64 CUDA, row-major."""
        import torch
        _check_dev(A, torch.float64, "A")
        n = A.shape[1] if n is None else n
        row_end = row_begin + A.shape[0] if row_end is None else row_end
        h = C.c_void_p()
        comm = refine_comm(rank, world, C.cast(C.c_char_p(nccl_id), C.c_void_p) if nccl_id else None)
        o = _opts(**opts)
        s = lib().refine_init_dense(C.byref(h), n, k, _ptr(A), A.stride(0), row_begin, row_end, float(shift),
                                    C.byref(comm), C.byref(o), _stream(stream))
        if s != REFINE_OK:
            raise RefineError(s, "refine_init_dense")
        return cls(h.value, n, k, row_end - row_begin, (A,), stream)

    @classmethod
    def csr(cls, row_ptr, col_idx, val, n: int, k: int, shift: float = 0.0, row_begin: int = 0,
            row_end: int | None = None, stream=None, rank: int = 0, world: int = 1,
            nccl_id: bytes | None = None, **opts) -> "Refiner":
        """refine_init_csr: int32 row_ptr (local rows + 1), int32 global col_idx, float64 val (CUDA)."""
        import torch
        _check_dev(row_ptr, torch.int32, "row_ptr")
        _check_dev(col_idx, torch.int32, "col_idx")
        _check_dev(val, torch.float64, "val")
        row_end = row_begin + row_ptr.numel() - 1 if row_end is None else row_end
        h = C.c_void_p()
        comm = refine_comm(rank, world, C.cast(C.c_char_p(nccl_id), C.c_void_p) if nccl_id else None)
        o = _opts(**opts)
        s = lib().refine_init_csr(C.byref(h), n, k, _ptr(row_ptr), _ptr(col_idx), _ptr(val), row_begin, row_end,
                                  float(shift), C.byref(comm), C.byref(o), _stream(stream))
        if s != REFINE_OK:
            raise RefineError(s, "refine_init_csr")
        return cls(h.value, n, k, row_end - row_begin, (row_ptr, col_idx, val), stream)

    # -- the sweep ---------------------------------------------------------------
    def refine_sweep(self, X, stats: bool = False):
        """One sweep on X (CUDA float64, n_loc x k) in place.  stats=True synchronises and
        returns (status, refine_sweep_stats); otherwise returns the enqueue status."""
        import torch
        _check_dev(X, torch.float64, "X")
        if stats:
            st = refine_sweep_stats()
            s = lib().refine_sweep(self._h, _ptr(X), C.byref(st))
            return s, st
        s = lib().refine_sweep(self._h, _ptr(X), None)
        if s != REFINE_OK:
            raise RefineError(s, "refine_sweep")
        return s

    def refine_sweep_host(self, X_in, X_out=None):
        """End-to-end sweep with host buffers (numpy float64 or CPU torch tensors)."""
        X_out = X_in if X_out is None else X_out
        st = refine_sweep_stats()
        pi = X_in.ctypes.data if hasattr(X_in, "ctypes") else X_in.data_ptr()
        po = X_out.ctypes.data if hasattr(X_out, "ctypes") else X_out.data_ptr()
        s = lib().refine_sweep_host(self._h, C.c_void_p(pi), C.c_void_p(po), C.byref(st))
        return s, st

    def refine_run(self, X, iters: int, tol: float):
        """Iterate sweeps until ||E_L||_F <= tol.  Returns (status, iters_done, last_stats)."""
        import torch
        _check_dev(X, torch.float64, "X")
        done = C.c_int32(0)
        st = refine_sweep_stats()
        s = lib().refine_run(self._h, _ptr(X), int(iters), float(tol), C.byref(done), C.byref(st))
        return s, done.value, st

    def refine_rayleigh_ritz(self, X):
        """Rayleigh-Ritz preprocessing (Sec. 3.4) on X in place: X <- X S with
        (X^T A X) S = (X^T X) S diag(ritz).  Returns (status, ritz as a numpy array, descending)."""
        import numpy as np
        import torch
        _check_dev(X, torch.float64, "X")
        ritz = np.zeros(self.k)
        s = lib().refine_rayleigh_ritz(self._h, _ptr(X), C.c_void_p(ritz.ctypes.data))
        return s, ritz

    def refine_reorthogonalize(self, X):
        """Cholesky-QR reorthogonalisation of X in place.  Returns (status, gram_dev before)."""
        import torch
        _check_dev(X, torch.float64, "X")
        gd = C.c_double(0.0)
        s = lib().refine_reorthogonalize(self._h, _ptr(X), C.byref(gd))
        return s, gd.value

    def refine_sweep_rr(self, X):
        """Rayleigh-Ritz, then one sweep with the E_L top block zero.
        Returns (status, refine_sweep_stats, ritz)."""
        import numpy as np
        import torch
        _check_dev(X, torch.float64, "X")
        ritz = np.zeros(self.k)
        st = refine_sweep_stats()
        s = lib().refine_sweep_rr(self._h, _ptr(X), C.byref(st), C.c_void_p(ritz.ctypes.data))
        return s, st, ritz

    def refine_get_status(self) -> int:
        return lib().refine_get_status(self._h)

    def refine_set_graph(self, enable: bool = True):
        s = lib().refine_set_graph(self._h, int(bool(enable)))
        if s != REFINE_OK:
            raise RefineError(s, "refine_set_graph")

    def kernels_per_sweep(self) -> int:
        return lib().refine_kernels_per_sweep(self._h)

    def refine_profile_begin(self, max_sweeps: int):
        s = lib().refine_profile_begin(self._h, int(max_sweeps))
        if s != REFINE_OK:
            raise RefineError(s, "refine_profile_begin")

    def refine_profile_end(self) -> tuple[dict, int]:
        """Returns ({kernel name: summed ms}, sweeps recorded)."""
        buf = (C.c_double * 32)()
        nk, ns = C.c_int32(0), C.c_int32(0)
        s = lib().refine_profile_end(self._h, buf, C.byref(nk), C.byref(ns))
        if s != REFINE_OK:
            raise RefineError(s, "refine_profile_end")
        names = [lib().refine_kernel_name(self._h, i).decode() for i in range(nk.value)]
        return {nm: buf[i] for i, nm in enumerate(names)}, ns.value

    def refine_debug_get(self, what: int, dst):
        s = lib().refine_debug_get(self._h, int(what), _ptr(dst))
        if s != REFINE_OK:
            raise RefineError(s, "refine_debug_get")
        return dst

    def debug(self, what: int, X_in=None):
        """Convenience: return the requested intermediate of the last sweep as a CUDA tensor."""
        import torch
        k, nl = self.k, self.n_loc
        shapes = {DBG_W: (nl, k), DBG_SIGMA: (k,), DBG_U: (k, k), DBG_L: (k, k), DBG_T: (k, k), DBG_D: (k,),
                  DBG_ALPHA: (k,), DBG_E11: (k, k), DBG_Y: (nl, k), DBG_STATS: (8,), DBG_SPMM: (9,)}
        if what == DBG_Y:
            dst = X_in.clone()
        else:
            dst = torch.empty(shapes[what], dtype=torch.float64, device="cuda")
        return self.refine_debug_get(what, dst)

    def refine_destroy(self):
        if self._h:
            lib().refine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.refine_destroy()
        except Exception:
            pass


def refine_nccl_id() -> bytes:
    buf = C.create_string_buffer(128)
    s = lib().refine_nccl_id(buf)
    if s != REFINE_OK:
        raise RefineError(s, "refine_nccl_id")
    return buf.raw


EXPORTED = ("refine_init_dense", "refine_init_csr", "refine_sweep", "refine_sweep_host", "refine_run",
            "refine_get_status", "refine_set_graph", "refine_kernels_per_sweep", "refine_destroy",
            "refine_status_string", "refine_nccl_id", "refine_debug_get", "refine_profile_begin",
            "refine_profile_end", "refine_kernel_name", "refine_halo_plan", "refine_rayleigh_ritz",
            "refine_sweep_rr", "refine_reorthogonalize")


def refine_halo_plan(world: int, rank: int, row_begin, row_end, col_lo, col_hi, cap: int = 64):
    """Host-only CSR halo plan of `rank` (see refine.h).  Returns (send, recv, halo_rows) with
    send/recv lists of (peer, first_row, count, offset)."""
    import numpy as np
    arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.int64)) for a in (row_begin, row_end, col_lo, col_hi)]
    send = np.zeros((cap, 4), dtype=np.int64)
    recv = np.zeros((cap, 4), dtype=np.int64)
    ns, nr, hr = C.c_int32(0), C.c_int32(0), C.c_int64(0)
    s = lib().refine_halo_plan(int(world), int(rank), *[a.ctypes.data for a in arrs], send.ctypes.data, C.byref(ns),
                               recv.ctypes.data, C.byref(nr), C.byref(hr), int(cap))
    if s != REFINE_OK:
        raise RefineError(s, "refine_halo_plan")
    return [tuple(map(int, r)) for r in send[:ns.value]], [tuple(map(int, r)) for r in recv[:nr.value]], hr.value
