"""Oracle pins for the Rayleigh-Ritz preprocessing (Sec. 3.4; SURVEY
NEXT-1) and the sweep that follows it (top block of E_L zero, beta = 0: PAPER.md:460, 921-926).

Pinned against things other than the oracle itself: exact eigenvectors of a Householder-product
matrix mixed by a known k x k matrix (closed form), scipy's generalized symmetric eigensolver
(an independent algorithm), numpy's eigh for the Jacobi kernel, the invariants the paper states
(Z^T Z = I, Z^T A Z = D~), span preservation, and the clustered-target behaviour of Table 6
(PAPER.md:1122-1142): plain refinement diverges, the preprocessed iteration converges."""
import numpy as np
import pytest
import scipy.linalg as sl

import oracle
import synth

U = 2.0 ** -53


def dense_op(p):
    return oracle.Operator(A=p.A.numpy(), shift=p.shift)


def test_jacobi_matches_eigh():
    rng = np.random.default_rng(3)
    for k in (1, 2, 5, 17, 40):
        C = rng.standard_normal((k, k))
        C = C + C.T
        Q, d = oracle.jacobi_eig(C)
        assert np.abs(np.sort(d) - np.linalg.eigvalsh(C)).max() <= 50 * k * U * np.linalg.norm(C)
        assert np.abs(Q.T @ Q - np.eye(k)).max() <= 50 * k * U
        assert np.abs(Q @ np.diag(d) @ Q.T - C).max() <= 50 * k * U * np.linalg.norm(C)


def test_jacobi_2x2_closed_form():
    a, b, c = 3.0, 1.5, -2.0
    Q, d = oracle.jacobi_eig(np.array([[a, b], [b, c]]))
    disc = np.sqrt(((a - c) / 2) ** 2 + b * b)
    assert np.allclose(np.sort(d), [(a + c) / 2 - disc, (a + c) / 2 + disc], rtol=0, atol=1e-15 * 4)


def test_rr_recovers_exact_eigenvectors():
    """X = V B with V exact eigenvectors (Householder-product truth) and B invertible: the Ritz pairs
    are exactly (lambda_j, +-v_j), ordered by descending lambda (reading RR3)."""
    p = synth.small_dense(200, 5, m=8, lam_target=np.array([7.0, -3.0, 9.0, 5.0, 6.0]), rest=1.0, seed=21)
    V = p.X.numpy()
    B = np.random.default_rng(4).standard_normal((5, 5)) + 3 * np.eye(5)
    s, Z, ritz = oracle.rayleigh_ritz(dense_op(p), V @ B)
    assert s == oracle.OK
    order = np.argsort(-p.lam_target)
    assert np.abs(ritz - p.lam_target[order]).max() <= 200 * U * 10
    Vs = V[:, order]
    sgn = np.sign(np.sum(Z * Vs, axis=0))
    assert np.abs(Z - Vs * sgn).max() <= 1e-12


def test_rr_invariants_and_pencil():
    """Z^T Z = I, Z^T A Z = diag(ritz), span(Z) = span(X), and the Ritz values
    equal the eigenvalues of the pencil (X^T A X, X^T X) from scipy (independent algorithm)."""
    p = synth.small_dense(300, 6, m=8, noise=1e-3, seed=8, signs=True)
    A, X = p.A.numpy(), p.X0.numpy()
    s, Z, ritz = oracle.rayleigh_ritz(dense_op(p), X)
    assert s == oracle.OK
    nA = np.abs(A).sum(1).max()
    assert np.abs(Z.T @ Z - np.eye(6)).max() <= 1e-13
    assert np.abs(Z.T @ A @ Z - np.diag(ritz)).max() <= 1e-12 * nA
    Px = X @ np.linalg.solve(X.T @ X, X.T)
    assert np.abs(Z @ Z.T - Px).max() <= 1e-12
    M = X.T @ A @ X
    ev = sl.eigh((M + M.T) / 2, X.T @ X, eigvals_only=True)
    assert np.abs(np.sort(ev)[::-1] - ritz).max() <= 1e-12 * nA
    assert np.all(np.diff(ritz) <= 0)


def test_rr_csr_matches_dense():
    q = synth.small_laplacian((15, 13), (1.0, 1.37), 4, noise=1e-3)
    rp, ci, v = q.row_ptr.numpy(), q.col_idx.numpy(), q.val.numpy()
    Ad = np.zeros((q.n, q.n))
    for i in range(q.n):
        Ad[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    s1, Z1, r1 = oracle.rayleigh_ritz(oracle.Operator(row_ptr=rp, col_idx=ci, val=v), q.X0.numpy())
    s2, Z2, r2 = oracle.rayleigh_ritz(oracle.Operator(A=Ad), q.X0.numpy())
    assert s1 == s2 == oracle.OK
    assert np.abs(r1 - r2).max() <= 1e-13 * np.abs(r2).max()
    sg = np.sign(np.sum(Z1 * Z2, axis=0))
    assert np.abs(Z1 - Z2 * sg).max() <= 1e-10


def test_rr_rank_deficient_is_invalid():
    p = synth.small_dense(100, 3, m=4, seed=2)
    X = p.X0.numpy().copy()
    X[:, 2] = X[:, 0]
    s, _, _ = oracle.rayleigh_ritz(dense_op(p), X)
    assert s == oracle.E_INVALID


def test_sweep_after_rr_has_zero_top_block():
    """After RR the sweep's top block is zero by construction; the remaining
    correction is the lower block v_ij / d_j (first-order power step)."""
    p = synth.small_dense(256, 4, m=8, noise=1e-5, seed=6)
    res, ritz = oracle.sweep_rr(dense_op(p), p.X0.numpy(), debug=True)
    assert res.status == oracle.OK and res.stats.delta_hits == 0
    D = res.debug
    k, n = p.k, p.n
    E, V, d = D["E"], D["V"], D["dtilde"]
    assert np.all(E[:k] == 0.0)                                    # e_ij = 0, i, j <= k
    assert np.array_equal(E[k:], V[k:] / d)                        # e_ij = v_ij / d_j, i > k (line 6)
    # independent route: X~ = Z' + H^ E~_L with H^ = I - Y T Y^T built explicitly (n x n), Z' the
    # RR output in the sweep's sign frame, E~_L = [0; V_2 D^{-1}] with V = H^T (A Z' - Z' D)
    Y, T, sig = D["Y"], D["T"], D["sigma"]
    H = np.eye(n) - Y @ T @ Y.T
    Zf = D["Z"] * sig
    A = p.A.numpy()
    Vref = H.T @ (A @ Zf - Zf * d)
    tolv = 64 * U * np.abs(A).sum(axis=1).max()                  # rounding of A Z' (no cancellation bound)
    assert np.abs(Vref[k:] - V[k:]).max() <= tolv
    El = np.vstack([np.zeros((k, k)), Vref[k:] / d])
    assert np.abs(D["Xtilde"] - (Zf + H @ El)).max() <= tolv / np.abs(d).min() + 1e-14


@pytest.mark.parametrize("gap", [1e-9, 1e-12])
def test_clustered_targets_rr_restores_convergence(gap):
    """Table 6 analogue: two targets closer than 1e-9 relative.  Plain
    refinement (Alg. 4, beta default) diverges; Rayleigh-Ritz + the top-zero sweep converges to
    the invariant subspace (sin angle <= 100 n u) and to ||E_L||_F <= 1e-13."""
    n, k = 256, 4
    p = synth.small_dense(n, k, m=8, lam_target=np.array([10.0, 9.0, 9.0 + 9.0 * gap, 8.0]), rest=1.0,
                          noise=1e-4, seed=5)
    op = dense_op(p)
    X, s, it, hist = oracle.run(op, p.X0.numpy(), 60, 1e-13)
    assert s == oracle.DIVERGED
    X = p.X0.numpy()
    for _ in range(40):
        res, ritz = oracle.sweep_rr(op, X)
        assert res.status == oracle.OK
        X = res.X
        if res.stats.corr_norm <= 1e-13:
            break
    assert res.stats.corr_norm <= 1e-13
    Xt = p.X.numpy()
    Q, _ = np.linalg.qr(X)
    assert np.linalg.norm(Xt - Q @ (Q.T @ Xt)) <= 100 * n * U
    assert np.abs(np.sort(ritz) - np.sort(p.lam_target)).max() <= 1e-13 * 10
