"""GPU parity of the Rayleigh-Ritz preprocessing (Sec. 3.4)
and of the preprocessed refinement iteration (RR + sweep with the E_L top block zero, PAPER.md:460,
921-926) against the oracle, through the C ABI (refine_rayleigh_ritz / refine_sweep_rr).

What is unique is compared element by element: the Ritz values (well conditioned) and, for
separated Ritz values, the Ritz vectors after the canonical signing (reading RR3).  For clustered
targets only the subspace is unique, so those cases compare projectors."""
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


def op_of(p):
    if p.kind == "dense":
        return oracle.Operator(A=p.A.cpu().numpy(), shift=p.shift)
    return oracle.Operator(row_ptr=p.row_ptr.numpy(), col_idx=p.col_idx.numpy(), val=p.val.numpy(), shift=p.shift)


def refiner(pkg, p, **kw):
    if p.kind == "dense":
        return pkg.Refiner.dense(p.A.cuda(), p.k, shift=p.shift, **kw)
    return pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, shift=p.shift, **kw)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def proj_diff(Z1, Z2):
    Q1, _ = np.linalg.qr(Z1)
    Q2, _ = np.linalg.qr(Z2)
    return float(np.linalg.norm(Q1 @ Q1.T @ Q2 - Q2))


CASES = [("dense", 300, 6), ("dense", 1100, 40), ("csr2d", 8, None), ("csr3d", 20, None), ("csr3d", 128, None)]


def make(kind, a, b):
    if kind == "dense":
        return synth.small_dense(a, b, m=8, noise=1e-3, seed=31, signs=True)
    if kind == "csr2d":
        return synth.small_laplacian((40, 37), (1.0, 1.37), a, noise=1e-4)
    return synth.small_laplacian((24, 22, 21), (1.0, 1.13, 1.29), a, noise=1e-4)


@pytest.mark.parametrize("kind,a,b", CASES)
def test_rr_parity(pkg, kind, a, b):
    p = make(kind, a, b)
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    s, ritz = R.refine_rayleigh_ritz(X)
    assert s == pkg.REFINE_OK
    so, Zo, ro = oracle.rayleigh_ritz(op_of(p), p.X0.numpy())
    assert so == oracle.OK
    scale = np.abs(ro).max()
    assert np.abs(ritz - ro).max() <= 1e-12 * scale
    Z = X.cpu().numpy()
    assert np.abs(Z.T @ Z - np.eye(p.k)).max() <= 1e-12
    assert proj_diff(Z, Zo) <= 1e-11
    gaps = np.abs(np.diff(ro))
    if gaps.min() > 1e-6 * scale:            # separated Ritz values: vectors are unique up to sign
        assert rel(Z, Zo) <= 1e-10


def test_rr_invariants_dense(pkg):
    p = synth.small_dense(512, 8, m=8, noise=1e-3, seed=4, signs=True)
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    s, ritz = R.refine_rayleigh_ritz(X)
    assert s == pkg.REFINE_OK
    Z, A = X.cpu().numpy(), p.A.numpy()
    assert np.abs(Z.T @ A @ Z - np.diag(ritz)).max() <= 1e-11 * np.abs(A).sum(1).max()
    assert np.all(np.diff(ritz) <= 0)


@pytest.mark.parametrize("kind,a,b", [("dense", 300, 6), ("csr2d", 8, None), ("csr3d", 20, None)])
def test_sweep_rr_one_step_parity(pkg, kind, a, b):
    p = make(kind, a, b)
    R = refiner(pkg, p)
    op = op_of(p)
    X = p.X0.cuda().clone()
    for t in range(3):
        xin = X.cpu().numpy()
        s, st, ritz = R.refine_sweep_rr(X)
        ref, ro = oracle.sweep_rr(op, xin)
        assert s == pkg.REFINE_OK and ref.status == oracle.OK
        assert rel(X.cpu().numpy(), ref.X) <= 1e-10, t
        assert abs(st.corr_norm - ref.stats.corr_norm) <= 1e-6 * ref.stats.corr_norm + 1e-12


@pytest.mark.parametrize("gap", [1e-9, 1e-12])
def test_clustered_targets_gpu(pkg, gap):
    """Table 6 analogue on the GPU: plain refinement diverges, the
    Rayleigh-Ritz iteration converges to ||E_L||_F <= 1e-13 and the invariant subspace."""
    n, k = 256, 4
    p = synth.small_dense(n, k, m=8, lam_target=np.array([10.0, 9.0, 9.0 + 9.0 * gap, 8.0]), rest=1.0,
                          noise=1e-4, seed=5)
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    s, it, st = R.refine_run(X, 60, 1e-13)
    assert s == pkg.REFINE_DIVERGED
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    for _ in range(40):
        s, st, ritz = R.refine_sweep_rr(X)
        assert s == pkg.REFINE_OK
        if st.corr_norm <= 1e-13:
            break
    assert st.corr_norm <= 1e-13
    assert proj_diff(X.cpu().numpy(), p.X.numpy()) <= 100 * n * U
    assert np.abs(np.sort(ritz) - np.sort(p.lam_target)).max() <= 1e-12


@pytest.mark.parametrize("kind,world", [("dense", 3), ("csr3d", 4)])
def test_rr_loopback(pkg, kind, world):
    p = make(kind, 300, 6) if kind == "dense" else make(kind, 20, None)
    X1, Xp = p.X0.cuda().clone(), p.X0.cuda().clone()
    s1, r1 = refiner(pkg, p).refine_rayleigh_ritz(X1)
    s2, r2 = refiner(pkg, p, world=world).refine_rayleigh_ritz(Xp)
    assert s1 == s2 == pkg.REFINE_OK
    assert np.abs(r1 - r2).max() <= 1e-13 * np.abs(r1).max()
    assert proj_diff(Xp.cpu().numpy(), X1.cpu().numpy()) <= 1e-12


def test_rr_rank_deficient(pkg):
    p = synth.small_dense(200, 3, m=4, seed=2)
    X = p.X0.cuda().clone()
    X[:, 2] = X[:, 0]
    s, _ = refiner(pkg, p).refine_rayleigh_ritz(X)
    assert s == pkg.REFINE_E_INVALID
