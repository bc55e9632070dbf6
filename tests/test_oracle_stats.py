"""Pins for the oracle's per-sweep statistics and the CSR operator norm, each against a value the
mathematics fixes independently of the oracle's own formulas:

* min_gap = min_{i != j} |d_j - d_i| (reported next to delta): at exact
  eigenvectors the Rayleigh quotients are the eigenvalues (eq. Rayleigh),
  so min_gap is the smallest gap of the chosen target eigenvalues.
* corr_norm = ||E~_L||_F: pinned in test_oracle_sweep.py
  (test_correction_against_exact_EL, against the exact E_L through an explicit H^) and here on
  the diagonal first-order case, where E~_L's lower block is eps (D_2 B_2 D_1^{-1} - B_2).
* ||A - shift I||_inf for CSR rows that store no diagonal (reading R4): the dense numpy norm.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle

U = 2.0 ** -53


def sym_with_spectrum(n, lam, seed):
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    q *= np.sign(np.diag(r))
    A = (q * lam) @ q.T
    return (A + A.T) / 2


@pytest.mark.parametrize("targets", [[10.0, 9.3, 7.0, 6.95], [-8.0, 8.0 - 1e-3, 5.5], [4.0, -4.25]])
def test_min_gap_is_smallest_target_gap(targets):
    n = 60
    k = len(targets)
    lam = np.concatenate([targets, np.linspace(-1.0, 1.0, n - k)])
    A = sym_with_spectrum(n, lam, 13)
    w, V = np.linalg.eigh(A)
    idx = [int(np.argmin(np.abs(w - t))) for t in targets]
    X = V[:, idx]
    r = oracle.sweep(oracle.Operator(A=A), X)
    assert r.status == oracle.OK
    t = np.asarray(targets)
    gaps = np.abs(t[:, None] - t[None, :])[~np.eye(k, dtype=bool)]
    assert abs(r.stats.min_gap - gaps.min()) <= 100 * n * U * np.abs(t).max()


def test_min_gap_single_column_is_zero():
    A = np.diag(np.linspace(5.0, 1.0, 10))
    r = oracle.sweep(oracle.Operator(A=A), np.eye(10, 1))
    assert r.status == oracle.OK and r.stats.min_gap == 0.0


def test_corr_norm_diagonal_first_order():
    """A = diag(lam), X^ = I_{n,k} + eps B with B's top block zero: the exact eigenvectors are
    I_{n,k}, so E_L's top block is O(eps^2) and its lower block is -eps B_2 to first order;
    E~_L (line 6) has lower block V_2 D~^{-1} = eps (D_2 B_2 D_1^{-1} - B_2) + O(eps^2)
    (first-order terms of eqs. V-def / Eoffdiag).  ||E~_L||_F must match that prediction."""
    n, k, eps = 50, 4, 1e-7
    lam = np.concatenate([[9.0, 8.0, 7.0, 6.0], np.linspace(-2.0, 2.0, n - k)])
    B = np.random.default_rng(8).standard_normal((n, k))
    B[:k] = 0.0
    X = np.eye(n, k) + eps * B
    r = oracle.sweep(oracle.Operator(A=np.diag(lam)), X, normalize=False)
    assert r.status == oracle.OK
    pred = eps * (lam[k:, None] * B[k:] / lam[None, :k] - B[k:])
    assert abs(r.stats.corr_norm - np.linalg.norm(pred)) <= 1e-4 * np.linalg.norm(pred)


def _csr_missing_diag():
    """Small symmetric CSR whose rows 3 and 7 store no diagonal entry (both triangles kept)."""
    rng = np.random.default_rng(3)
    n = 12
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(i, min(n, i + 3)):
            A[i, j] = A[j, i] = rng.uniform(-2.0, 2.0)
    A[3, 3] = 0.0
    A[7, 7] = 0.0
    M = sp.csr_matrix(A)
    M.eliminate_zeros()
    M.sort_indices()
    assert M[3, 3] == 0.0 and 3 not in M.indices[M.indptr[3]:M.indptr[4]]
    return A, M


@pytest.mark.parametrize("shift", [0.0, 0.75, -3.5])
def test_csr_norm_inf_with_missing_diagonal(shift):
    A, M = _csr_missing_diag()
    op = oracle.Operator(row_ptr=M.indptr, col_idx=M.indices, val=M.data, shift=shift)
    ref = np.abs(A - shift * np.eye(A.shape[0])).sum(axis=1).max()
    assert abs(op.norm_inf() - ref) <= 4 * A.shape[0] * U * ref
    X = np.random.default_rng(4).standard_normal((A.shape[0], 3))
    W = op.apply(X)
    bound = 4 * 13 * U * (np.abs(A) @ np.abs(X) + abs(shift) * np.abs(X))
    assert np.all(np.abs(W - (A @ X - shift * X)) <= bound)


def test_rel_resid_uses_shifted_norm_with_missing_diagonal():
    """rel_resid = ||R||_F / ||A - shift I||_inf (reading R4): dense and CSR with
    the same matrix and shift report the same statistic."""
    A, M = _csr_missing_diag()
    X = np.random.default_rng(5).standard_normal((A.shape[0], 2))
    rd = oracle.sweep(oracle.Operator(A=A, shift=0.75), X)
    rc = oracle.sweep(oracle.Operator(row_ptr=M.indptr, col_idx=M.indices, val=M.data, shift=0.75), X)
    assert rd.status == rc.status == oracle.OK
    assert abs(rd.stats.rel_resid - rc.stats.rel_resid) <= 1e-13 * rd.stats.rel_resid
