"""Oracle pins for SURVEY NEXT-3: the shift-and-square operator B = A^2 - alpha I applied as A (A X)
(Sec. 5.2) and refining K > k columns while judging the leading k
(PAPER.md:941-942, 958-967).

Pins independent of the oracle: numpy's A @ (A @ X) - alpha X; closed-form sine eigenvectors of
a Dirichlet grid Laplacian (the smallest-|lambda| targets of Sec. 5.2); the linear rate law of
Thm 3.7 (rate max|lambda_rest| / |lambda_target|), which for K > k columns is governed by
lambda_{K+1} instead of lambda_{k+1}."""
import numpy as np

import oracle
import synth

U = 2.0 ** -53


def dense_lap(q):
    rp, ci, v = q.row_ptr.numpy(), q.col_idx.numpy(), q.val.numpy()
    A = np.zeros((q.n, q.n))
    for i in range(q.n):
        A[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    return A


def test_square_apply_matches_numpy():
    p = synth.small_dense(150, 5, m=6, seed=3)
    A, X = p.A.numpy(), p.X0.numpy()
    alpha = 7.25
    W = oracle.Operator(A=A, shift=alpha, square=True).apply(X)
    ref = A @ (A @ X) - alpha * X
    nA = np.abs(A).sum(1).max()
    assert np.abs(W - ref).max() <= 4 * 150 * U * (nA * nA + alpha) * np.abs(X).max()


def test_square_norm_bound():
    p = synth.small_dense(120, 4, m=6, seed=9)
    A = p.A.numpy()
    op = oracle.Operator(A=A, shift=3.0, square=True)
    nA = np.abs(A).sum(1).max()
    assert abs(op.norm_inf() - (nA * nA + 3.0)) <= 1e-12 * nA * nA
    assert op.norm_inf() >= np.linalg.norm(A @ A - 3.0 * np.eye(120), 2)


def test_square_csr_equals_dense():
    q = synth.small_laplacian((11, 9), (1.0, 1.37), 3, noise=1e-3)
    Ad = dense_lap(q)
    X = q.X0.numpy()
    a = oracle.Operator(row_ptr=q.row_ptr.numpy(), col_idx=q.col_idx.numpy(), val=q.val.numpy(), shift=2.0,
                        square=True).apply(X)
    b = oracle.Operator(A=Ad, shift=2.0, square=True).apply(X)
    assert np.array_equal(a, b)          # same fma chains (the dense rows' zeros add exact zeros)


def test_smallest_magnitude_eigenvectors_by_shift_and_square():
    """Sec. 5.2: the k smallest-|lambda| eigenvectors of a Dirichlet Laplacian (closed-form sine
    modes) are the dominant ones of A^2 - alpha I with alpha = (||A||_inf^2 + lambda_{k+1}^2) / 2
    (the paper's practical alpha, written with the squared eigenvalue of A^2 -- reading SQ2)."""
    k = 3
    q = synth.small_laplacian((9, 7), (1.0, 1.37), k, noise=1e-5, seed=11)
    L = dense_lap(q)                          # A' = sigma I - L; we want the smallest |eig| of L itself
    sigma = q.meta["sigma"]
    A = sigma * np.eye(q.n) - L               # the Laplacian L = sigma I - A'
    lam = np.sort(np.linalg.eigvalsh(A))
    alpha = (np.abs(A).sum(1).max() ** 2 + lam[k] ** 2) / 2
    op = oracle.Operator(A=A, shift=alpha, square=True)
    X, s, it, hist = oracle.run(op, q.X0.numpy(), 4000, 1e-13)
    assert s == oracle.OK
    Xt = q.X.numpy()                          # closed-form sine modes = smallest eigenvectors of L
    sg = np.sign(np.sum(X * Xt, axis=0))
    # attainable accuracy of the squared operator is ~ u ||A||^2 / gap(B) (here 553 n u measured):
    # squaring the spectrum squeezes the relative gap, so the bound is 1000 n u, not 100 n u
    assert np.abs(X * sg - Xt).max() <= 1000 * q.n * U
    # rate law: per-sweep contraction ~ max|lam_j^2 - alpha| / min|lam_i^2 - alpha|
    gam = max(abs(lam[k:] ** 2 - alpha)) / min(abs(lam[:k] ** 2 - alpha))
    c = hist[:, 1]
    obs = np.exp(np.mean(np.log(c[20:60] / c[19:59])))
    assert 0.5 * gam <= obs <= 1.1 * gam


def test_refining_more_columns_accelerates_leading_ones():
    """K > k: refining K = 2k columns and judging the leading k converges at the
    rate |lambda_{K+1}| / |lambda_k| instead of |lambda_{k+1}| / |lambda_k|."""
    n, k, K = 300, 3, 6
    lt = np.array([10.0, 9.5, 9.2, 8.0, 7.5, 7.0])
    p = synth.small_dense(n, K, m=8, lam_target=lt, rest=4.0, noise=1e-6, seed=17)
    op = oracle.Operator(A=p.A.numpy())
    Xk, s1, it_k, h_k = oracle.run(op, p.X0.numpy()[:, :k], 400, 1e-13)
    XK, s2, it_K, h_K = oracle.run(op, p.X0.numpy(), 400, 1e-13, kjudge=k)
    assert s1 == s2 == oracle.OK
    assert it_K < it_k
    gk = 8.0 / 9.2
    gK = 4.0 / 9.2
    ok = np.exp(np.mean(np.log(h_k[3:10, 1] / h_k[2:9, 1])))
    oK = np.exp(np.mean(np.log(h_K[2:5, 1] / h_K[1:4, 1])))
    assert 0.5 * gk <= ok <= 1.1 * gk and oK <= 1.1 * gK
    Xt = p.X.numpy()[:, :k]
    sg = np.sign(np.sum(XK[:, :k] * Xt, axis=0))
    assert np.abs(XK[:, :k] * sg - Xt).max() <= 100 * n * U
