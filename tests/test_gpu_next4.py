"""GPU parity for SURVEY NEXT-4 (refine_run robustness policies) against the oracle through the
C ABI: Cholesky-QR reorthogonalisation (refine_reorthogonalize), the Gram-deviation
statistic, the residual stopping criterion, the reorthogonalisation policy and
the divergence-triggered switch to Rayleigh-Ritz."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_23778_b200 as p
    from paper_2602_23778_b200 import build
    build.build()
    p.lib()
    assert torch.cuda.is_available()
    return p


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_reorthogonalize_parity(pkg, kind):
    if kind == "dense":
        p = synth.small_dense(700, 12, m=8, noise=1e-3, seed=9)
        R = pkg.Refiner.dense(p.A.cuda(), p.k)
    else:
        p = synth.small_laplacian((24, 22, 21), (1.0, 1.13, 1.29), 20, noise=1e-3)
        R = pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k)
    rng = np.random.default_rng(1)
    X0 = p.X0.numpy() @ (np.eye(p.k) + 0.05 * rng.standard_normal((p.k, p.k)))
    X = torch.from_numpy(X0).cuda()
    s, gd = R.refine_reorthogonalize(X)
    so, Zo, gdo = oracle.reorthogonalize(X0)
    assert s == pkg.REFINE_OK and so == oracle.OK
    assert abs(gd - gdo) <= 1e-12 * gdo
    Z = X.cpu().numpy()
    assert rel(Z, Zo) <= 1e-12
    assert np.abs(Z.T @ Z - np.eye(p.k)).max() <= 1e-13


def test_gram_dev_statistic(pkg):
    p = synth.small_dense(400, 6, m=8, noise=1e-3, seed=4)
    R = pkg.Refiner.dense(p.A.cuda(), p.k, reorth_tol=1.0)
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, st = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(oracle.Operator(A=p.A.numpy()), xin, want_gram=True)
    assert abs(st.gram_dev - ref.stats.gram_dev) <= 1e-12 + 1e-10 * ref.stats.gram_dev
    s, st = pkg.Refiner.dense(p.A.cuda(), p.k).refine_sweep(p.X0.cuda().clone(), stats=True)
    assert st.gram_dev == -1.0


def test_residual_stopping(pkg):
    p = synth.small_dense(256, 4, m=8, noise=1e-5, seed=3)
    op = oracle.Operator(A=p.A.numpy())
    R = pkg.Refiner.dense(p.A.cuda(), p.k, resid_tol=1e-9)
    X = p.X0.cuda().clone()
    s, it, st = R.refine_run(X, 50, 0.0)
    Xo, so, ito, ho = oracle.run_policy(op, p.X0.numpy(), 50, 0.0, resid_tol=1e-9)
    assert s == pkg.REFINE_OK and so == oracle.OK and it == ito
    assert st.rel_resid <= 1e-9
    assert rel(X.cpu().numpy(), Xo) <= 1e-9


def test_reorth_policy(pkg):
    n, k = 300, 5
    p = synth.small_dense(n, k, m=8, noise=1e-7, seed=7, fp32=False)
    X0 = p.X0.numpy() @ (np.eye(k) + 3e-3 * np.random.default_rng(2).standard_normal((k, k)))
    op = oracle.Operator(A=p.A.numpy())
    R = pkg.Refiner.dense(p.A.cuda(), k, reorth_tol=1e-6)
    X = torch.from_numpy(X0).cuda()
    s, it, st = R.refine_run(X, 200, 1e-13)
    Xo, so, ito, ho = oracle.run_policy(op, X0, 200, 1e-13, reorth_tol=1e-6)
    assert s == pkg.REFINE_OK and so == oracle.OK and abs(it - ito) <= 1
    Xg, Xt = X.cpu().numpy(), p.X.numpy()
    sg = np.sign(np.sum(Xg * Xt, 0))
    assert np.abs(Xg * sg - Xt).max() <= 100 * n * U
    assert np.abs(Xg.T @ Xg - np.eye(k)).max() <= 1e-12


@pytest.mark.parametrize("world", [2, 3])
def test_reorth_policy_row_partition(pkg, world):
    """The reorthogonalisation policy at world > 1 (loopback ranks; the host reads the device gate
    after each sweep): the same iteration count as the oracle's policy loop and the 100 n u accuracy."""
    n, k = 300, 5
    p = synth.small_dense(n, k, m=8, noise=1e-7, seed=7, fp32=False)
    X0 = p.X0.numpy() @ (np.eye(k) + 3e-3 * np.random.default_rng(2).standard_normal((k, k)))
    op = oracle.Operator(A=p.A.numpy())
    R = pkg.Refiner.dense(p.A.cuda(), k, reorth_tol=1e-6, world=world)
    X = torch.from_numpy(X0).cuda()
    s, it, st = R.refine_run(X, 200, 1e-13)
    Xo, so, ito, ho = oracle.run_policy(op, X0, 200, 1e-13, reorth_tol=1e-6)
    assert s == pkg.REFINE_OK and so == oracle.OK and abs(it - ito) <= 1
    Xg, Xt = X.cpu().numpy(), p.X.numpy()
    sg = np.sign(np.sum(Xg * Xt, 0))
    assert np.abs(Xg * sg - Xt).max() <= 100 * n * U
    assert np.abs(Xg.T @ Xg - np.eye(k)).max() <= 1e-12


def test_divergence_falls_back_to_rayleigh_ritz(pkg):
    n, k = 256, 4
    p = synth.small_dense(n, k, m=8, lam_target=np.array([10.0, 9.0, 9.0 + 9e-12, 8.0]), rest=1.0,
                          noise=1e-4, seed=5)
    R = pkg.Refiner.dense(p.A.cuda(), k)
    X = p.X0.cuda().clone()
    s, it, st = R.refine_run(X, 80, 1e-13)
    assert s == pkg.REFINE_DIVERGED
    R = pkg.Refiner.dense(p.A.cuda(), k, rr_fallback=True)
    X = p.X0.cuda().clone()
    s, it, st = R.refine_run(X, 80, 1e-13)
    assert s == pkg.REFINE_OK and st.corr_norm <= 1e-13
    Q, _ = np.linalg.qr(X.cpu().numpy())
    Xt = p.X.numpy()
    assert np.linalg.norm(Xt - Q @ (Q.T @ Xt)) <= 100 * n * U


def test_normalize_false_with_closed_reorth_gate(pkg):
    """refine_run with normalize=False and a reorthogonalisation threshold that never triggers:
    the gated Cholesky-QR step (enqueued every sweep behind the device gate) must leave X alone,
    so the run equals the same run without the policy, bit for bit."""
    p = synth.small_dense(600, 8, m=8, noise=1e-4, seed=4)
    Ra = pkg.Refiner.dense(p.A.cuda(), p.k, normalize=False)
    Rb = pkg.Refiner.dense(p.A.cuda(), p.k, normalize=False, reorth_tol=10.0)
    Xa, Xb = p.X0.cuda().clone(), p.X0.cuda().clone()
    sa, ia, _ = Ra.refine_run(Xa, 6, 0.0)
    sb, ib, _ = Rb.refine_run(Xb, 6, 0.0)
    assert sa == sb == pkg.REFINE_MAXITER and ia == ib == 6
    assert torch.equal(Xa, Xb)


@pytest.mark.parametrize("normalize", [True, False])
def test_rank_deficient_leaves_X_unchanged(pkg, normalize):
    """Rayleigh-Ritz and Cholesky QR on a rank-deficient X return REFINE_E_INVALID and leave X
    untouched (refine.h), whether or not the step normalises."""
    p = synth.small_dense(500, 6, m=8, seed=12)
    R = pkg.Refiner.dense(p.A.cuda(), p.k, normalize=normalize)
    X0 = p.X0.cuda().clone()
    X0[:, 3] = X0[:, 1]
    X = X0.clone()
    s, _ = R.refine_rayleigh_ritz(X)
    assert s == pkg.REFINE_E_INVALID and torch.equal(X, X0)
    s, _ = R.refine_reorthogonalize(X)
    assert s == pkg.REFINE_E_INVALID and torch.equal(X, X0)


def test_guard_window_out_of_range_rejected(pkg):
    p = synth.small_dense(200, 4, m=4, seed=1)
    for w in (5, -1):
        with pytest.raises(pkg.RefineError) as ei:
            pkg.Refiner.dense(p.A.cuda(), p.k, guard_window=w)
        assert ei.value.status == pkg.REFINE_E_INVALID
