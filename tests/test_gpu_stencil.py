"""The stencil SpMM (spmm_stencil.cuh): S1 for CSR matrices whose nonzeros couple grid points only
with themselves and their axis neighbours (the configs' Laplacians), X staged by 4-D TMA boxes.

Checked through the C ABI against the oracle (P3: W bit-identical -- the same fma chain in CSR
order -- and one-step parity P1) on 2-D and 3-D grids, every column-block width (k = 8 .. 128),
partial tiles, the shift path, and against the gather kernel (REFINE_SPMM=gather) bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import compare_sweep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_23778_b200 as p
    from paper_2602_23778_b200 import build
    build.build()
    p.lib()
    assert torch.cuda.is_available()
    return p


@pytest.fixture(autouse=True)
def force_stencil(monkeypatch):
    """By default the library takes the stencil SpMM for 3-D grids with k >= 64 and 2-D grids with k a
    multiple of 32 (where it measured faster); REFINE_SPMM=stencil makes every eligible matrix take it,
    so each case below exercises it (small grids: most CTAs get an empty slab range)."""
    monkeypatch.setenv("REFINE_SPMM", "stencil")


def refiner(pkg, p, **kw):
    return pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, shift=p.shift, **kw)


def op_of(p):
    return oracle.Operator(row_ptr=p.row_ptr.numpy(), col_idx=p.col_idx.numpy(), val=p.val.numpy(), shift=p.shift)


def geometry(pkg, R):
    return R.debug(pkg.DBG_SPMM).cpu().numpy()


CASES = [((64, 61), (1.0, 1.37), 8), ((64, 61), (1.0, 1.37), 32), ((64, 61), (1.0, 1.37), 128),
         ((200, 7), (1.0, 1.37), 16), ((24, 22, 21), (1.0, 1.13, 1.29), 8), ((24, 22, 21), (1.0, 1.13, 1.29), 32),
         ((24, 22, 21), (1.0, 1.13, 1.29), 64), ((24, 22, 21), (1.0, 1.13, 1.29), 128),
         ((37, 29, 11), (1.0, 1.13, 1.29), 48), ((17, 15, 13), (1.0, 1.13, 1.29), 16),
         # tiles away from every x / y face: slab blocks whose rows are all canonical (the no-code-word path)
         ((72, 40, 10), (1.0, 1.13, 1.29), 32), ((72, 40, 10), (1.0, 1.13, 1.29), 128), ((600, 9), (1.0, 1.37), 32)]


@pytest.mark.parametrize("dims,coeffs,k", CASES)
def test_stencil_w_bitwise_and_one_step(pkg, dims, coeffs, k):
    p = synth.small_laplacian(dims, coeffs, k)
    R = refiner(pkg, p)
    geo = geometry(pkg, R)
    assert geo[0] == 1.0, f"stencil SpMM not selected: {geo}"
    nx, ny, nz = geo[5:8]
    assert nx * ny * nz == p.n and nx == dims[0]
    op = op_of(p)
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, st = R.refine_sweep(X, stats=True)
    assert s == pkg.REFINE_OK
    ref = oracle.sweep(op, xin, debug=True)
    assert np.array_equal(R.debug(pkg.DBG_W).cpu().numpy() * ref.debug["sigma"], ref.debug["W"])
    compare_sweep(X.cpu().numpy(), ref, st, k=p.k, normA=op.norm_inf())


def test_stencil_with_shift(pkg):
    """Sec. 5.1: L with shift sigma (B = L - sigma I = -A'), W = fma(-shift, x, chain)."""
    p = synth.small_laplacian((30, 29, 9), (1.0, 1.13, 1.29), 16)
    rp, ci, v = p.row_ptr.numpy(), p.col_idx.numpy(), p.val.numpy()
    diag = ci == np.repeat(np.arange(p.n), np.diff(rp))
    p.val = torch.from_numpy(np.where(diag, p.meta["sigma"] - v, -v))
    p.shift = p.meta["sigma"]
    R = refiner(pkg, p)
    assert geometry(pkg, R)[0] == 1.0
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, st = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(op_of(p), xin, debug=True)
    assert s == pkg.REFINE_OK
    assert np.array_equal(R.debug(pkg.DBG_W).cpu().numpy() * ref.debug["sigma"], ref.debug["W"])
    compare_sweep(X.cpu().numpy(), ref, st, k=p.k, normA=op_of(p).norm_inf())


@pytest.mark.parametrize("dims,coeffs,k", [((64, 61), (1.0, 1.37), 32), ((24, 22, 21), (1.0, 1.13, 1.29), 128)])
def test_stencil_equals_gather_kernel(pkg, dims, coeffs, k, monkeypatch):
    p = synth.small_laplacian(dims, coeffs, k)
    Xa, Xb = p.X0.cuda().clone(), p.X0.cuda().clone()
    Ra = refiner(pkg, p)
    assert geometry(pkg, Ra)[0] == 1.0
    Ra.refine_sweep(Xa)
    monkeypatch.setenv("REFINE_SPMM", "gather")
    Rb = refiner(pkg, p)
    assert geometry(pkg, Rb)[0] == 0.0
    Rb.refine_sweep(Xb)
    assert torch.equal(Ra.debug(pkg.DBG_W), Rb.debug(pkg.DBG_W))
    d = float((Xa - Xb).abs().max())
    assert d <= 1e-13, d


def test_stencil_graph_and_determinism(pkg):
    p = synth.small_laplacian((40, 33, 17), (1.0, 1.13, 1.29), 64)
    R = refiner(pkg, p)
    Xa, Xb = p.X0.cuda().clone(), p.X0.cuda().clone()
    R.refine_sweep(Xa)
    R.refine_sweep(Xa)
    R.refine_set_graph(True)
    R.refine_sweep(Xb)
    R.refine_sweep(Xb)
    R.refine_set_graph(False)
    assert torch.equal(Xa, Xb)


def test_non_stencil_matrix_takes_gather_kernel(pkg):
    """A nonzero outside the axis-neighbour set (here a coupling across the grid) disables the
    stencil path; the gather kernel keeps W bit-identical."""
    import scipy.sparse as sp
    p = synth.small_laplacian((30, 29), (1.0, 1.37), 16)
    A = sp.csr_matrix((p.val.numpy(), p.col_idx.numpy(), p.row_ptr.numpy()), shape=(p.n, p.n)).tolil()
    A[3, 500] = A[500, 3] = 1e-3
    A = A.tocsr()
    A.sort_indices()
    import dataclasses
    q = dataclasses.replace(p, row_ptr=torch.from_numpy(A.indptr.astype(np.int32)),
                            col_idx=torch.from_numpy(A.indices.astype(np.int32)), val=torch.from_numpy(A.data))
    R = refiner(pkg, q)
    assert geometry(pkg, R)[0] == 0.0
    X = q.X0.cuda().clone()
    xin = X.cpu().numpy()
    R.refine_sweep(X)
    ref = oracle.sweep(op_of(q), xin, debug=True)
    assert np.array_equal(R.debug(pkg.DBG_W).cpu().numpy() * ref.debug["sigma"], ref.debug["W"])


def test_stencil_default_policy_fullsize(pkg, monkeypatch):
    """Default policy at full size: cfg5 (3-D, k = 128) and cfg4 (2-D, k = 32) take the stencil SpMM
    (their parity runs in test_gpu_fullsize), with one CTA per SM and 128-point line segments on the
    2-D grid."""
    monkeypatch.delenv("REFINE_SPMM")
    for name, want in (("cfg4", 1.0), ("cfg5", 1.0)):
        p = synth.make_config(name, device="cuda")
        R = pkg.Refiner.csr(p.row_ptr, p.col_idx, p.val, p.n, p.k)
        geo = geometry(pkg, R)
        print(name, "S1 geometry [stencil, R, L, nq, grid, nx, ny, nz, gatherR]", geo.tolist())
        assert geo[0] == want
        if name == "cfg4":
            assert geo[1] == 128 and geo[2] == 1
        del R, p
        torch.cuda.empty_cache()
