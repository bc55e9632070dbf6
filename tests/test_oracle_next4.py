"""Oracle pins for SURVEY NEXT-4 (robustness policies of refine_run): Cholesky-QR
reorthogonalisation, the residual stopping criterion and the
divergence-triggered switch to Rayleigh-Ritz preprocessing.

Independent pins: the QR factorisation (X = Q R with R upper triangular, positive diagonal ->
Cholesky QR returns Q exactly), numpy Gram matrices and residuals, and the clustered-target case
where plain refinement diverges (Table 6 analogue)."""
import numpy as np

import oracle
import synth

U = 2.0 ** -53


def test_reorthogonalize_returns_q_of_qr():
    rng = np.random.default_rng(5)
    n, k = 400, 7
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    R = np.triu(rng.standard_normal((k, k))) + 3 * np.eye(k)
    R[np.diag_indices(k)] = np.abs(R[np.diag_indices(k)])
    X = Q @ R
    s, Z, gd = oracle.reorthogonalize(X)
    assert s == oracle.OK
    assert np.abs(Z - Q).max() <= 1e-13
    assert abs(gd - np.abs(X.T @ X - np.eye(k)).max()) <= 1e-12 * gd
    assert np.abs(Z.T @ Z - np.eye(k)).max() <= 1e-14


def test_reorthogonalize_rank_deficient():
    X = np.random.default_rng(1).standard_normal((50, 3))
    X[:, 1] = 2 * X[:, 0]
    assert oracle.reorthogonalize(X)[0] == oracle.E_INVALID


def test_sweep_reports_gram_deviation():
    p = synth.small_dense(256, 4, m=8, noise=1e-3, seed=12)
    X = p.X0.numpy()
    res = oracle.sweep(oracle.Operator(A=p.A.numpy()), X, want_gram=True)
    assert abs(res.stats.gram_dev - np.abs(X.T @ X - np.eye(4)).max()) <= 1e-14


def test_residual_stopping_criterion():
    """refine_run stops at the first sweep whose input has ||A X - X D||_F / ||A||_inf <= resid_tol."""
    p = synth.small_dense(256, 4, m=8, noise=1e-5, seed=3)
    op = oracle.Operator(A=p.A.numpy())
    A = p.A.numpy()
    tol = 1e-9
    X, s, it, hist = oracle.run_policy(op, p.X0.numpy(), 50, 0.0, resid_tol=tol)
    assert s == oracle.OK and hist[-1, 0] <= tol and np.all(hist[:-1, 0] > tol)
    Xin, _, _, _ = oracle.run_policy(op, p.X0.numpy(), it - 1, 0.0)    # the last sweep's input
    d = np.sum(Xin * (A @ Xin), 0) / np.sum(Xin * Xin, 0)
    res = np.linalg.norm(A @ Xin - Xin * d) / np.abs(A).sum(1).max()
    assert abs(res - hist[-1, 0]) <= 1e-6 * res


def test_divergence_switches_to_rayleigh_ritz():
    """'If ||E_L||_F grows rapidly ... switch to preprocessing'.  Clustered targets
    (gap 1e-12): the plain run trips the guard; with rr_fallback it converges."""
    n, k = 256, 4
    p = synth.small_dense(n, k, m=8, lam_target=np.array([10.0, 9.0, 9.0 + 9e-12, 8.0]), rest=1.0,
                          noise=1e-4, seed=5)
    op = oracle.Operator(A=p.A.numpy())
    X, s, it, hist = oracle.run_policy(op, p.X0.numpy(), 80, 1e-13)
    assert s == oracle.DIVERGED
    X, s, it, hist = oracle.run_policy(op, p.X0.numpy(), 80, 1e-13, rr_fallback=True)
    assert s == oracle.OK and hist[-1, 2] == 1 and hist[0, 2] == 0
    Q, _ = np.linalg.qr(X)
    Xt = p.X.numpy()
    assert np.linalg.norm(Xt - Q @ (Q.T @ Xt)) <= 100 * n * U


def test_reorthogonalisation_policy():
    """An input with orthogonality loss (non-orthogonal mixing inside the target subspace) triggers
    the Cholesky-QR step after the first sweep; the run still converges to 100 n u."""
    n, k = 300, 5
    p = synth.small_dense(n, k, m=8, noise=1e-7, seed=7, fp32=False)
    rng = np.random.default_rng(2)
    X0 = p.X0.numpy() @ (np.eye(k) + 3e-3 * rng.standard_normal((k, k)))
    op = oracle.Operator(A=p.A.numpy())
    X, s, it, hist = oracle.run_policy(op, X0, 200, 1e-13, reorth_tol=1e-6)
    assert s == oracle.OK
    res = oracle.sweep(op, X, want_gram=True)
    assert res.stats.gram_dev <= 1e-10
    Xt = p.X.numpy()
    sg = np.sign(np.sum(X * Xt, 0))
    assert np.abs(X * sg - Xt).max() <= 100 * n * U
