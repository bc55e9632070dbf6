"""Seeded synthetic inputs for the refinement sweep -- the ONLY module shared by the
oracle side (tests, cpu baseline) and the CUDA side (tests, bench).

It holds none of the method's arithmetic: it builds the matrices A, the known
eigenvectors X and the perturbed starting blocks X0 of BASELINE.json's configs.
Recipe:

* dense configs (stand-ins for the paper's gallery('randsvd') matrices,
  PAPER.md:977-978): A = Q diag(lam) Q^T with Q = H_1 ... H_m a product of m
  seeded Householder reflectors H_r = I - 2 v v^T / (v^T v), v ~ N(0, I_n);
  targets at positions 1..k so the truth is X = Q[:, :k]; A symmetrised as
  (A + A^T)/2 so it is exactly symmetric.
* sparse configs (stand-ins for the SuiteSparse matrices):
  anisotropic Dirichlet grid Laplacians L (5-/7-point, unscaled stencil,
  lexicographic order, x fastest), A' = sigma I - L with sigma = 4 * sum(c);
  the k smallest-mu modes of L are closed-form sine products, which are the
  k largest eigenpairs of A'.
* X0 = X + N(0, s^2) noise (row-major draw), rounded to fp32 for the dense
  configs as BASELINE.json says (stand-in for single-precision eigs,
  PAPER.md:943-948).

Random draws: numpy Generator(PCG64(seed)); seed_A = c, seed_X = 100 + c.  Draw
order for rng_A: reflector vectors v_1..v_m (n normals each), target magnitudes
(if random), the n-k other eigenvalues, target signs (if random).  rng_X: the
n x k noise, row-major.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch


@dataclass
class Problem:
    name: str
    n: int
    k: int
    sweeps: int
    kind: str                      # "dense" | "csr"
    shift: float = 0.0
    # dense
    A: Optional[torch.Tensor] = None          # n x n float64 row-major (device of choice)
    # csr (both triangles, sorted columns, int32 indices)
    row_ptr: Optional[torch.Tensor] = None
    col_idx: Optional[torch.Tensor] = None
    val: Optional[torch.Tensor] = None
    lam: Optional[np.ndarray] = None          # full spectrum of the operator (dense: exact values used)
    lam_target: Optional[np.ndarray] = None   # eigenvalues of the k targets, column order
    X: Optional[torch.Tensor] = None          # truth n x k
    X0: Optional[torch.Tensor] = None         # start n x k
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.val.numel()) if self.kind == "csr" else self.n * self.n

    def gamma(self) -> float:
        """max_{i>k}|lam_i| / min_{j<=k}|lam_j|."""
        rest = np.delete(self.lam, np.arange(self.k)) if self.kind == "dense" else self.meta["lam_rest_absmax"]
        rmax = float(np.max(np.abs(rest))) if self.kind == "dense" else float(rest)
        return rmax / float(np.min(np.abs(self.lam_target)))


# --------------------------------------------------------------------------- dense

def householder_vectors(rng: np.random.Generator, n: int, m: int) -> np.ndarray:
    return rng.standard_normal((m, n))


def apply_reflectors(V: torch.Tensor, M: torch.Tensor) -> torch.Tensor:
    """Return H_1 ... H_m M for reflectors H_r = I - 2 v_r v_r^T/(v_r^T v_r) (rows of V)."""
    for r in range(V.shape[0] - 1, -1, -1):
        v = V[r]
        M = M - (2.0 / torch.dot(v, v)) * torch.outer(v, v @ M)
    return M


def dense_from_reflectors(V: torch.Tensor, lam: torch.Tensor) -> torch.Tensor:
    """A = Q diag(lam) Q^T, Q = H_1...H_m, built by two-sided reflector updates, symmetrised."""
    A = torch.diag(lam)
    for r in range(V.shape[0] - 1, -1, -1):       # A <- H_r A H_r, innermost reflector first
        v = V[r]
        c = 2.0 / torch.dot(v, v)
        A.addr_(v, v @ A, alpha=-c)                # H A
        A.addr_(A @ v, v, alpha=-c)                # (H A) H
    A.add_(A.T.clone()).mul_(0.5)                  # exact symmetry: fl(a+b) = fl(b+a)
    return A


def make_dense(name: str, n: int, k: int, m: int, lam_target: np.ndarray | None, target_mag: tuple | None,
               rest: float, noise: float, sweeps: int, seed: int, device="cpu", signs: bool = False,
               geometric: float | None = None, fp32: bool = True) -> Problem:
    rng = np.random.Generator(np.random.PCG64(seed))
    V = householder_vectors(rng, n, m)
    if lam_target is None:
        if geometric is not None:
            mags = 100.0 * geometric ** np.arange(k)
        else:
            mags = rng.uniform(target_mag[0], target_mag[1], size=k)
    else:
        mags = np.asarray(lam_target, dtype=np.float64)
    lam_rest = rng.uniform(-rest, rest, size=n - k)
    sg = np.where(rng.random(k) < 0.5, -1.0, 1.0) if signs else np.ones(k)
    lt = mags * sg
    lam = np.concatenate([lt, lam_rest])
    dev = torch.device(device)
    Vt = torch.from_numpy(V).to(dev)
    A = dense_from_reflectors(Vt, torch.from_numpy(lam).to(dev))
    E = torch.zeros(n, k, dtype=torch.float64, device=dev)
    E[torch.arange(k), torch.arange(k)] = 1.0
    X = apply_reflectors(Vt, E)                   # X = Q I_{n,k}
    rngx = np.random.Generator(np.random.PCG64(100 + seed))
    nz = torch.from_numpy(rngx.standard_normal((n, k)) * noise).to(dev)
    X0 = X + nz
    if fp32:
        X0 = X0.float().double()
    return Problem(name=name, n=n, k=k, sweeps=sweeps, kind="dense", A=A.contiguous(), lam=lam,
                   lam_target=lt, X=X.contiguous(), X0=X0.contiguous(), meta={"m": m, "seed": seed})


# --------------------------------------------------------------------------- sparse

def laplacian_modes(dims, coeffs, k):
    """k smallest eigenvalues mu of the anisotropic Dirichlet Laplacian and their mode
    indices p (1-based per axis), sorted ascending (ties broken by lexicographic p)."""
    dims = list(dims)
    # mu = sum_d c_d 4 sin^2(p_d pi / (2 (N_d + 1)));  candidate p_d <= k suffices
    cand = [np.arange(1, min(N, k + 1) + 1) for N in dims]
    mus = [c * 4.0 * np.sin(p * np.pi / (2.0 * (N + 1))) ** 2 for c, p, N in zip(coeffs, cand, dims)]
    grids = np.meshgrid(*[np.arange(len(c)) for c in cand], indexing="ij")
    tot = sum(mu[g] for mu, g in zip(mus, grids)).ravel()
    idx = np.stack([g.ravel() for g in grids], axis=1)
    order = np.lexsort(tuple(idx[:, d] for d in range(len(dims) - 1, -1, -1)) + (tot,))
    order = order[:k + 1]
    P = np.stack([cand[d][idx[order, d]] for d in range(len(dims))], axis=1)
    return tot[order], P


def sine_modes(dims, P, device="cpu") -> torch.Tensor:
    """Closed-form eigenvectors of the Dirichlet Laplacian: product over axes of
    sqrt(2/(N+1)) sin(p pi i/(N+1)), i = 1..N, lexicographic with axis 0 fastest."""
    dev = torch.device(device)
    k = P.shape[0]
    X = None
    for d, N in enumerate(dims):
        i = torch.arange(1, N + 1, dtype=torch.float64, device=dev)
        p = torch.from_numpy(P[:, d].astype(np.float64)).to(dev)
        f = math.sqrt(2.0 / (N + 1)) * torch.sin(torch.outer(i, p) * (math.pi / (N + 1)))  # N x k
        # new index = i_d * (size so far) + old index  (axis 0 fastest)
        X = f if X is None else (f.reshape(N, 1, k) * X.reshape(1, -1, k)).reshape(-1, k)
    return X.contiguous()


def laplacian_csr(dims, coeffs):
    """CSR of A' = sigma I - L, sigma = 4 sum(c): diag 2 sum(c), neighbours +c_d, sorted columns."""
    dims = list(dims)
    n = int(np.prod(dims))
    strides = [int(np.prod(dims[:d])) for d in range(len(dims))]
    coords = np.indices(dims[::-1]).reshape(len(dims), -1)[::-1]  # coords[d] for lexicographic index, axis 0 fastest
    cols, vals = [], []
    diag = 2.0 * sum(coeffs)
    # neighbours in ascending column order: -axis_{D-1} ... -axis_0, self, +axis_0 ... +axis_{D-1}
    offs = []
    for d in range(len(dims) - 1, -1, -1):
        offs.append((d, -1))
    offs.append((None, 0))
    for d in range(len(dims)):
        offs.append((d, +1))
    rows_all = np.arange(n, dtype=np.int64)
    entries_r, entries_c, entries_v = [], [], []
    for d, s in offs:
        if d is None:
            entries_r.append(rows_all); entries_c.append(rows_all); entries_v.append(np.full(n, diag))
        else:
            ok = (coords[d] + s >= 0) & (coords[d] + s < dims[d])
            r = rows_all[ok]
            entries_r.append(r); entries_c.append(r + s * strides[d]); entries_v.append(np.full(r.size, float(coeffs[d])))
    r = np.concatenate(entries_r); c = np.concatenate(entries_c); v = np.concatenate(entries_v)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr.astype(np.int32), c.astype(np.int32), v.astype(np.float64), 4.0 * sum(coeffs)


def make_laplacian(name, dims, coeffs, k, noise, sweeps, seed, device="cpu") -> Problem:
    rp, ci, v, sigma = laplacian_csr(dims, coeffs)
    n = int(np.prod(dims))
    mu, P = laplacian_modes(dims, coeffs, k)
    dev = torch.device(device)
    X = sine_modes(dims, P[:k], dev)
    rngx = np.random.Generator(np.random.PCG64(100 + seed))
    X0 = X + torch.from_numpy(rngx.standard_normal((n, k)) * noise).to(dev)
    lam_t = sigma - mu[:k]
    # largest |eigenvalue| of A' outside the targets is sigma - mu_{k+1} (all eigenvalues are in (0, sigma))
    return Problem(name=name, n=n, k=k, sweeps=sweeps, kind="csr", shift=0.0,
                   row_ptr=torch.from_numpy(rp).to(dev), col_idx=torch.from_numpy(ci).to(dev),
                   val=torch.from_numpy(v).to(dev), lam=None, lam_target=lam_t, X=X, X0=X0.contiguous(),
                   meta={"dims": list(dims), "coeffs": list(coeffs), "sigma": sigma, "modes": P[:k].tolist(),
                         "mu": mu[:k].tolist(), "lam_rest_absmax": sigma - mu[k], "seed": seed})


# --------------------------------------------------------------------------- configs

CONFIGS = ("cfg1", "cfg2", "cfg2b", "cfg3", "cfg4", "cfg5")


def make_config(name: str, device="cpu", n: int | None = None) -> Problem:
    """BASELINE.json configs[0..4] (cfg1..cfg5) plus cfg2b (cfg2 with ratio 5/9 over the
    targets, reading R12).  `n` scales the dense configs down for CPU tests."""
    if name == "cfg1":
        return make_dense("cfg1", n or 256, 4, 8, [10.0, 9.0, 8.0, 7.0], None, 1.0, 1e-6, 10, 1, device)
    if name == "cfg2":
        return make_dense("cfg2", n or 4096, 16, 32, None, None, 50.0, 1e-5, 20, 2, device, signs=True,
                          geometric=0.95)
    if name == "cfg2b":
        return make_dense("cfg2b", n or 4096, 16, 32, None, None, 50.0, 1e-5, 20, 2, device, signs=True,
                          geometric=(5.0 / 9.0) ** (1.0 / 15.0))
    if name == "cfg3":
        return make_dense("cfg3", n or 32768, 64, 64, None, (90.0, 100.0), 80.0, 1e-6, 15, 3, device, signs=True)
    if name == "cfg4":
        return make_laplacian("cfg4", (1024, 1021), (1.0, 1.37), 32, 1e-6, 10, 4, device)
    if name == "cfg5":
        return make_laplacian("cfg5", (160, 160, 160), (1.0, 1.13, 1.29), 128, 1e-6, 10, 5, device)
    raise KeyError(name)


def small_laplacian(dims, coeffs, k, noise=1e-6, seed=7, device="cpu") -> Problem:
    """Scaled-down sparse config with the same structure (tests)."""
    return make_laplacian(f"lap{'x'.join(map(str, dims))}", dims, coeffs, k, noise, 10, seed, device)


def small_dense(n, k, m=8, lam_target=None, rest=1.0, noise=1e-6, seed=11, device="cpu", signs=False,
                target_mag=(90.0, 100.0), fp32=True) -> Problem:
    return make_dense(f"dense{n}x{k}", n, k, m, lam_target, target_mag if lam_target is None else None, rest,
                      noise, 10, seed, device, signs=signs, fp32=fp32)
