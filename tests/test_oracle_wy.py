"""Pins for the oracle's WY construction (Alg. 1-3) against
hand traces, the algorithms' own Ensure lines and textbook identities -- none of these
re-types the oracle's code: they check products formed independently with numpy."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def orthonormal(n, k, seed):
    """Random orthonormal n x k block from numpy's Householder QR (LAPACK), independent of the oracle."""
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, k)))
    return q * np.sign(np.diag(r))


def H_of(Y, T):
    n = Y.shape[0]
    return np.eye(n) - Y @ T @ Y.T


def test_hand_traces_modified_lu():
    g = json.load(open(os.path.join(GOLD, "spec_hand_traces.json")))
    for case in g["modified_lu"]:
        Y, Uf, sig, st = oracle.modified_lu(np.array(case["Q"]))
        assert st == oracle.OK
        assert np.array_equal(sig, case["sigma"])
        assert np.array_equal(Uf, case["U"])
        assert np.array_equal(Y, case["Y"])


def test_hand_traces_compact_wy_lu_and_alg1():
    g = json.load(open(os.path.join(GOLD, "spec_hand_traces.json")))
    for case in g["compact_wy_lu"]:
        Y, T, sig, Uf, st = oracle.compact_wy_lu(np.array(case["Q"]))
        assert st == oracle.OK
        assert np.array_equal(T, case["T"])
        H = H_of(Y, T)
        assert np.array_equal(H, case["H"])
        assert np.array_equal(H[:, :1], case["H_e1"])
    for case in g["compact_wy"]:
        Y, T, st = oracle.compact_wy(np.array(case["Q"]))
        assert st == oracle.OK
        assert np.array_equal(Y, case["Y"]) and np.array_equal(T, case["T"])
        assert np.array_equal(H_of(Y, T), case["H"])


@pytest.mark.parametrize("n,k,seed", [(20, 5, 0), (64, 16, 1), (300, 40, 2), (33, 32, 3)])
def test_modified_lu_ensure(n, k, seed):
    """Alg. 2 Ensure: Q - Sigma = Y U, Y unit lower, U upper, |u_jj| >= 1."""
    Q = orthonormal(n, k, seed)
    Y, Uf, sig, st = oracle.modified_lu(Q)
    assert st == oracle.OK
    S = np.zeros((n, k)); S[np.arange(k), np.arange(k)] = sig
    assert np.linalg.norm(Q - S - Y @ Uf) <= 50 * k * U * np.linalg.norm(Q)
    assert np.allclose(np.triu(Y[:k], 1), 0) and np.all(np.diag(Y[:k]) == 1.0)
    assert np.allclose(np.tril(Uf, -1), 0)
    assert np.all(np.abs(np.diag(Uf)) >= 1.0 - 1e-15)   # |q_jj - sigma_j| >= 1 by the sign choice
    assert set(np.unique(sig)) <= {-1.0, 1.0}


@pytest.mark.parametrize("n,k,seed", [(30, 4, 4), (200, 24, 5), (129, 64, 6)])
def test_compact_wy_lu_ballard(n, k, seed):
    """Alg. 3: I - Y T Y^T is orthogonal and maps I_{n,k} to Q Sigma (reading R2: the
    Ensure line's 'Q' holds as Q Sigma); after X <- X Sigma, H^T X = [I; 0]."""
    Q = orthonormal(n, k, seed)
    Q[:, ::2] *= -1.0      # make Sigma mixed
    Y, T, sig, Uf, st = oracle.compact_wy_lu(Q)
    assert st == oracle.OK
    H = H_of(Y, T)
    assert np.linalg.norm(H.T @ H - np.eye(n)) <= 1e-13
    assert np.linalg.norm(H[:, :k] - Q * sig) <= 1e-13
    if np.any(sig < 0):   # the misprinted Ensure line fails whenever Sigma != I
        assert np.linalg.norm(H[:, :k] - Q) > 1.0
    Iq = np.zeros((n, k)); Iq[:k] = np.eye(k)
    assert np.linalg.norm(H.T @ (Q * sig) - Iq) <= 1e-13
    # T = -U Sigma Y1^{-T}  <=>  T Y1^T = -U Sigma   (independent check by multiplication)
    assert np.linalg.norm(T @ Y[:k].T + Uf * sig) <= 1e-13 * max(1.0, np.linalg.norm(Uf))


@pytest.mark.parametrize("n,k,seed", [(40, 6, 7), (150, 20, 8)])
def test_flip_makes_alg1_equal_alg3(n, k, seed):
    """After the one-time flip X <- X Sigma, modified LU returns sigma' = +1, Y' = Y,
    U' = U Sigma, and Alg. 1 builds the same H."""
    Q = orthonormal(n, k, seed)
    Y, T, sig, Uf, st = oracle.compact_wy_lu(Q)
    Qf = Q * sig
    Y2, U2, sig2, st2 = oracle.modified_lu(Qf)
    assert st2 == oracle.OK and np.all(sig2 == 1.0)
    assert np.array_equal(Y2, Y)
    assert np.array_equal(U2, Uf * sig)
    Y1, T1, st1 = oracle.compact_wy(Qf)
    assert st1 == oracle.OK
    assert np.linalg.norm(H_of(Y1, T1) - H_of(Y, T)) <= 1e-12


def test_alg1_fails_on_identity_block():
    """Alg. 1 needs Y_1 nonsingular: Q = I_{n,k} gives Y_1 = 0."""
    Q = np.zeros((6, 2)); Q[0, 0] = Q[1, 1] = 1.0
    _, _, st = oracle.compact_wy(Q)
    assert st == oracle.E_ZERO_PIVOT
    Y, T, sig, Uf, st = oracle.compact_wy_lu(Q)     # Alg. 3 works: sigma = -1, H I = -I
    assert st == oracle.OK and np.all(sig == -1.0)
    assert np.allclose(H_of(Y, T)[:, :2], -Q, atol=0)


@pytest.mark.parametrize("transpose", [False, True])
def test_apply_h_matches_explicit(transpose):
    """H B = B - Y(T(Y^T B)) equals the explicit n x n product."""
    n, k, m = 90, 7, 5
    Q = orthonormal(n, k, 9)
    Y, T, sig, _, _ = oracle.compact_wy_lu(Q)
    B = np.random.default_rng(10).standard_normal((n, m))
    H = H_of(Y, T)
    ref = (H.T if transpose else H) @ B
    got = oracle.apply_h(Y, T, B, transpose)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(B)
    back = oracle.apply_h(Y, T, oracle.apply_h(Y, T, B, False), True)   # H^T H = I
    assert np.linalg.norm(back - B) <= 1e-13 * np.linalg.norm(B)
