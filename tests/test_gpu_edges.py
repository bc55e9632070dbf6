"""Degenerate shapes and argument errors through the C ABI: the smallest problems the method
admits (k = 1, n = 2), k = n - 1 (a single row below the top block) up to k = 128 = KMAX, the
same for CSR, and the statuses of invalid or unsupported shapes."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_23778_b200 as p
    from paper_2602_23778_b200 import build
    build.build()
    p.lib()
    return p


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,k", [(2, 1), (5, 4), (33, 32), (64, 63), (129, 128)])
def test_dense_k_is_n_minus_1(pkg, n, k):
    p = synth.small_dense(n, k, m=4, seed=n, signs=True)
    R = pkg.Refiner.dense(p.A.cuda(), k)
    op = oracle.Operator(A=p.A.numpy())
    X = p.X0.cuda().clone()
    for t in range(3):
        xin = X.cpu().numpy()
        s, st = R.refine_sweep(X, stats=True)
        ref = oracle.sweep(op, xin)
        assert s == pkg.REFINE_OK and ref.status == oracle.OK
        assert rel(X.cpu().numpy(), ref.X) <= TOL, t
        assert st.flipped == ref.stats.flipped


def test_csr_k_is_n_minus_1(pkg):
    p = synth.small_laplacian((5, 4), (1.0, 1.37), 19, noise=1e-5, seed=3)
    R = pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k)
    op = oracle.Operator(row_ptr=p.row_ptr.numpy(), col_idx=p.col_idx.numpy(), val=p.val.numpy())
    X = p.X0.cuda().clone()
    for t in range(3):
        xin = X.cpu().numpy()
        s, _ = R.refine_sweep(X, stats=True)
        ref = oracle.sweep(op, xin)
        assert s == pkg.REFINE_OK and ref.status == oracle.OK
        assert rel(X.cpu().numpy(), ref.X) <= TOL, t


@pytest.mark.parametrize("n,k,status", [(100, 0, "REFINE_E_INVALID"), (100, 100, "REFINE_E_INVALID"),
                                        (100, 150, "REFINE_E_INVALID"), (300, 129, "REFINE_E_UNSUPPORTED")])
def test_invalid_shapes(pkg, n, k, status):
    A = torch.eye(n, dtype=torch.float64, device="cuda")
    with pytest.raises(pkg.RefineError) as ei:
        pkg.Refiner.dense(A, k)
    assert ei.value.status == getattr(pkg, status)


def test_wrong_tensor_kinds(pkg):
    A = torch.eye(64, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        pkg.Refiner.dense(A.float(), 4)                 # FP32 A
    with pytest.raises(TypeError):
        pkg.Refiner.dense(A.t()[:, :32], 4)             # non-contiguous
    with pytest.raises(TypeError):
        pkg.Refiner.dense(A.cpu(), 4)                   # host tensor on the device entry point


@pytest.mark.parametrize("n,k,opt", [(33, 32, {"mixed": 2}), (129, 128, {"mixed": 2}), (129, 128, {"emul": True}),
                                     (17, 16, {"emul": True})])
def test_tensor_core_paths_k_is_n_minus_1(pkg, n, k, opt):
    """NEXT-2 (bf16x3) and INT8 passes with a single row below the top block."""
    p = synth.small_dense(n, k, m=4, seed=n + 7, signs=True)
    R = pkg.Refiner.dense(p.A.cuda(), k, **opt)
    op = oracle.Operator(A=p.A.numpy())
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, _ = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(op, xin)
    assert s == pkg.REFINE_OK and ref.status == oracle.OK
    sig = np.where(np.sum(ref.X * xin, axis=0) < 0, -1.0, 1.0)
    corr = np.linalg.norm(ref.X - xin * sig)
    # mixed: 1e-2 of the correction (tests/test_gpu_mixed.py); emul: the FP64 bar
    tol = 1e-2 * corr + 1e-10 * np.linalg.norm(ref.X) if "mixed" in opt else 1e-10 * np.linalg.norm(ref.X)
    assert np.linalg.norm(X.cpu().numpy() - ref.X) <= tol


def _csr_of(A):
    rp, ci, v = [0], [], []
    for i in range(A.shape[0]):
        nz = np.nonzero(A[i])[0]
        ci.extend(nz.tolist())
        v.extend(A[i, nz].tolist())
        rp.append(len(ci))
    return (torch.tensor(rp, dtype=torch.int32), torch.tensor(ci, dtype=torch.int32),
            torch.tensor(v, dtype=torch.float64))


@pytest.mark.parametrize("k", [8, 32])
def test_csr_empty_rows(pkg, k):
    """CSR rows without any nonzero (row / column zeroed, first and last rows included): W's rows
    are exactly zero there and the sweep matches the oracle."""
    p = synth.small_dense(400, k, m=8, seed=k, signs=True)
    A = p.A.numpy().copy()
    A[np.abs(A) < 1e-3] = 0.0                           # sparse-ish, symmetric
    for r in (0, 17, 250, 399):
        A[r, :] = 0.0
        A[:, r] = 0.0
    rp, ci, v = _csr_of(A)
    R = pkg.Refiner.csr(rp.cuda(), ci.cuda(), v.cuda(), 400, k)
    op = oracle.Operator(row_ptr=rp.numpy(), col_idx=ci.numpy(), val=v.numpy())
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, _ = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(op, xin)
    assert s == pkg.REFINE_OK and ref.status == oracle.OK
    assert rel(X.cpu().numpy(), ref.X) <= TOL


@pytest.mark.parametrize("n,k,shift", [(256, 4, 0.0), (1000, 16, 0.0), (3001, 64, 0.75), (777, 13, 0.0)])
def test_fused_split_k_finish_matches_w_finish(pkg, n, k, shift, monkeypatch):
    """Dense S1's split-K fix-up fused into the GEMM (the last CTA of a row tile sums the partials,
    applies the shift and writes the alpha/g slot; REFINE_WFUSE=1) against the separate w_finish kernel
    (REFINE_WFUSE=0): W bit-identical (same split order), X~ equal to rounding, both at oracle parity."""
    p = synth.small_dense(n, k, m=8, seed=n, signs=True)
    op = oracle.Operator(A=p.A.numpy(), shift=shift)
    outs = {}
    for fuse in ("1", "0"):
        monkeypatch.setenv("REFINE_WFUSE", fuse)
        R = pkg.Refiner.dense(p.A.cuda(), k, shift=shift)
        X = p.X0.cuda().clone()
        xin = X.cpu().numpy()
        s, st = R.refine_sweep(X, stats=True)
        assert s == pkg.REFINE_OK
        outs[fuse] = (R.debug(pkg.DBG_W).cpu().numpy(), X.cpu().numpy())
        ref = oracle.sweep(op, xin)
        assert rel(X.cpu().numpy(), ref.X) <= TOL, fuse
    assert np.array_equal(outs["1"][0], outs["0"][0])
    assert rel(outs["1"][1], outs["0"][1]) <= 1e-13
