"""GPU parity of Alg. 4 line 6's delta / beta branch (PAPER.md:439-447 second case, beta choices
PAPER.md:453-460; reading R5: the test |d_j - d_i| <= delta is inclusive, R6: beta = -x_i^T x_j / 2
by default, 0 under beta_zero).

No BASELINE config produces a delta hit, so the branch is exercised on constructed inputs whose
Rayleigh-quotient gaps sit far from the threshold delta = c ||A - shift I||_inf u on either side
(so that both sides take the same decision whatever the summation order):

* an exact tie: A diagonal with lambda_1 = lambda_2 and identical perturbations of the two tied
  columns -> d_1 == d_2 bit for bit on both sides;
* near ties on a dense Q diag(lambda) Q^T: target gaps 2^-50 lambda (hit), 2^-40 lambda (no hit, just
  above delta: ill-conditioned, so X is compared within u ||A||_inf / gap) and 2^-16 lambda (no hit,
  well separated: the 1e-10 bar), start noise 1e-10 so the Rayleigh quotients stay within
  O(eps^2 ||A||) of lambda;
* the degenerate sine modes (p, q) / (q, p) of an isotropic Dirichlet Laplacian (CSR): the two
  modes of a pair have the same eigenvalue, their computed Rayleigh quotients differ by rounding.

Each case runs with beta_zero off and on, single rank and loopback ranks (world 2 and 3), and checks
delta_hits (> 0 and equal to the oracle's), E_11 through refine_debug_get(DBG_E11) within 1e-12,
and one-step parity (whole block and per row block) within the north_star's 1e-10."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import compare_sweep, cond_tol

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


def _exact_tie(n=300, k=4):
    lam = np.concatenate([[4.0, 4.0, 3.0, 2.5][:k], np.linspace(-1.0, 1.0, n - k)])
    A = np.diag(lam)
    X = np.eye(n, k)
    rng = np.random.default_rng(1)
    rows = rng.choice(np.arange(k, n), size=40, replace=False)
    pert = 1e-3 * rng.standard_normal(40)
    X[rows, 0] = pert
    X[rows, 1] = pert                        # identical perturbations -> identical Rayleigh quotients
    for j in range(2, k):
        X[rng.choice(np.arange(k, n), size=10, replace=False), j] = 1e-3 * rng.standard_normal(10)
    return A, X


def _near_tie(g, n=520, k=4, seed=5):
    p = synth.small_dense(n, k, m=8, lam_target=np.array([10.0, 9.0, 9.0 + 9.0 * g, 8.0]), rest=1.0,
                          noise=1e-10, seed=seed, fp32=False)
    return p.A.numpy(), p.X0.numpy()


def _laplacian_pairs(N=40, k=8):
    return synth.small_laplacian((N, N), (1.0, 1.0), k, noise=1e-10, seed=3)


def _refiner(pkg, A=None, k=None, p=None, world=1, beta_zero=False):
    if p is None:
        return pkg.Refiner.dense(torch.from_numpy(A).cuda(), k, world=world, beta_zero=beta_zero)
    return pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, world=world,
                           beta_zero=beta_zero)


def _check(pkg, R, op, X0, k, beta_zero, expect_hits):
    """One sweep on the GPU and in the oracle from the same input."""
    X = torch.from_numpy(np.ascontiguousarray(X0)).cuda()
    s, st = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(op, X0, beta_zero=beta_zero, debug=True)
    assert s == pkg.REFINE_OK and ref.status == oracle.OK, (s, ref.status)
    d = ref.debug["dtilde"]
    delta = 10.0 * op.norm_inf() * U
    gaps = np.abs(d[:, None] - d[None, :])[~np.eye(k, dtype=bool)]
    # the decision is robust: every gap is at least 4x away from delta on its side
    assert np.all((gaps <= delta / 4) | (gaps >= 4 * delta)), (gaps.min(), delta)
    assert ref.stats.delta_hits == int((gaps <= delta).sum())
    if expect_hits:
        assert ref.stats.delta_hits > 0
    else:
        assert ref.stats.delta_hits == 0
    # Without a hit, E_ij = V_ij / gap amplifies the O(u ||A||) rounding of V by 1 / gap: a gap just
    # above delta (2^-40 lambda here) makes one-step agreement to 1e-10 impossible for ANY two
    # summation orders, so the bar is max(1e-10, u ||A||_inf / gap) there; the branch
    # decision itself (delta_hits, which formula each entry used) must still agree exactly.
    ctol = cond_tol(ref, op.norm_inf())
    compare_sweep(X.cpu().numpy(), ref, st, k=k, where=f"beta_zero={beta_zero}", tol=ctol, elem_tol=ctol,
                  corr_rel=max(1e-6, ctol), corr_abs=max(1e-9, k * ctol))
    E11 = R.debug(pkg.DBG_E11).cpu().numpy()
    Eo = ref.debug["E"][:k]
    assert np.abs(E11 - Eo).max() <= max(1e-12, ctol * max(1.0, np.abs(Eo).max())), np.abs(E11 - Eo).max()
    if expect_hits:
        hit = np.abs(d[:, None] - d[None, :]) <= delta
        np.fill_diagonal(hit, False)
        if beta_zero:
            assert np.all(E11[hit] == 0.0)
        else:
            # beta_ij = -x^_i^T x^_j / 2 of the flipped input
            Xf = X0 * ref.debug["sigma"]
            G = Xf.T @ Xf
            assert np.abs(E11[hit] + G[hit] / 2).max() <= 1e-15 + 1e-13 * np.abs(G[hit]).max()
    return st, ref


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("beta_zero", [False, True])
def test_delta_exact_tie_dense(pkg, world, beta_zero):
    A, X0 = _exact_tie()
    k = X0.shape[1]
    R = _refiner(pkg, A=A, k=k, world=world, beta_zero=beta_zero)
    st, ref = _check(pkg, R, oracle.Operator(A=A), X0, k, beta_zero, True)
    assert ref.debug["dtilde"][0] == ref.debug["dtilde"][1]
    assert st.delta_hits == 2 and st.min_gap == 0.0


@pytest.mark.parametrize("g,hit", [(2.0 ** -50, True), (2.0 ** -40, False), (2.0 ** -16, False)])
@pytest.mark.parametrize("beta_zero", [False, True])
@pytest.mark.parametrize("world", [1, 2])
def test_delta_near_tie_dense_both_sides(pkg, g, hit, beta_zero, world):
    A, X0 = _near_tie(g)
    k = X0.shape[1]
    R = _refiner(pkg, A=A, k=k, world=world, beta_zero=beta_zero)
    _check(pkg, R, oracle.Operator(A=A), X0, k, beta_zero, hit)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("beta_zero", [False, True])
def test_delta_degenerate_laplacian_modes_csr(pkg, world, beta_zero):
    p = _laplacian_pairs()
    R = _refiner(pkg, p=p, world=world, beta_zero=beta_zero)
    op = oracle.Operator(row_ptr=p.row_ptr.numpy(), col_idx=p.col_idx.numpy(), val=p.val.numpy())
    st, ref = _check(pkg, R, op, p.X0.numpy(), p.k, beta_zero, True)
    assert st.delta_hits == 6               # the pairs (1,2)/(2,1), (1,3)/(3,1), (2,3)/(3,2)


def test_delta_run_matches_oracle_iterations(pkg):
    """Three sweeps through the branch: trajectory parity (independent runs) on the exact tie."""
    A, X0 = _exact_tie()
    R = _refiner(pkg, A=A, k=X0.shape[1])
    op = oracle.Operator(A=A)
    X = torch.from_numpy(X0.copy()).cuda()
    Xo = X0.copy()
    for t in range(3):
        s, st = R.refine_sweep(X, stats=True)
        r = oracle.sweep(op, Xo)
        Xo = r.X
        assert s == pkg.REFINE_OK and r.status == oracle.OK
        assert st.delta_hits == r.stats.delta_hits == 2
        diff = np.linalg.norm(X.cpu().numpy() - Xo) / np.linalg.norm(Xo)
        assert diff <= 1e-10, (t, diff)
