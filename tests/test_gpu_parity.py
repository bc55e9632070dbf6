"""GPU parity: the CUDA sweep (through the C ABI) against the oracle, element by element.

North_star bar: per-sweep relative Frobenius difference <= 1e-10 (one-step parity P1:
the oracle consumes the GPU's own input X_t); converged eigenvector error <= 100 n u.
Kernel-level (P3): CSR W bit-identical; dense W within gamma_n |A||X|; k x k factors
<= 1e-13 relative.  Sizes span several tiles and ragged tails; the full BASELINE sizes
run in test_gpu_fullsize.py."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
U = 2.0 ** -53
TOL = 1e-10


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_23778_b200 as p
    from paper_2602_23778_b200 import build
    build.build()
    p.lib()
    assert torch.cuda.is_available()
    return p


from parity_util import compare_sweep, rel  # noqa: E402


def op_of(p):
    if p.kind == "dense":
        return oracle.Operator(A=p.A.cpu().numpy(), shift=p.shift)
    return oracle.Operator(row_ptr=p.row_ptr.cpu().numpy(), col_idx=p.col_idx.cpu().numpy(),
                           val=p.val.cpu().numpy(), shift=p.shift)


def refiner(pkg, p, **kw):
    if p.kind == "dense":
        return pkg.Refiner.dense(p.A.cuda(), p.k, shift=p.shift, **kw)
    return pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, shift=p.shift, **kw)


def one_step(pkg, p, sweeps, R=None, op=None, stats_tol=1e-8):
    """P1: at every sweep t run the oracle on the GPU's X_t and compare with X_{t+1} (the whole
    block, each of its two row blocks per column, and the statistics incl. min_gap)."""
    R = R or refiner(pkg, p)
    op = op or op_of(p)
    X = p.X0.cuda().clone()
    worst = 0.0
    for t in range(sweeps):
        xin = X.cpu().numpy()
        s, st = R.refine_sweep(X, stats=True)
        ref = oracle.sweep(op, xin, debug=True)
        assert s == pkg.REFINE_OK and ref.status == oracle.OK, (t, s, ref.status)
        e = compare_sweep(X.cpu().numpy(), ref, st, k=p.k, stats_tol=stats_tol, where=f"sweep {t}",
                          normA=op.norm_inf())
        worst = max(worst, e)
    return worst, X


# ------------------------------------------------------------------------------ dense

def test_cfg1_one_step_parity(pkg):
    p = synth.make_config("cfg1")
    worst, _ = one_step(pkg, p, p.sweeps)
    print(f"cfg1 worst one-step rel diff {worst:.3e}")


def test_cfg1_trajectory_parity_and_convergence(pkg):
    """P2 (independent trajectories) and the converged accuracy gate <= 100 n u."""
    p = synth.make_config("cfg1")
    R = refiner(pkg, p)
    op = op_of(p)
    X = p.X0.cuda().clone()
    Xo = p.X0.numpy().copy()
    for t in range(p.sweeps):
        R.refine_sweep(X)
        Xo = oracle.sweep(op, Xo).X
        assert rel(X.cpu().numpy(), Xo) <= TOL, t
    s, it, st = R.refine_run(X, 30, 1e-15)
    Xt = p.X.numpy()
    Xg = X.cpu().numpy()
    sg = np.sign(np.sum(Xg * Xt, axis=0))
    assert np.linalg.norm(Xg * sg - Xt, axis=0).max() <= 100 * p.n * U


@pytest.mark.parametrize("n,k,shift", [(200, 1, 0.0), (300, 3, 0.0), (517, 5, 0.5), (1000, 12, 0.0),
                                       (777, 16, 0.0), (1200, 33, 0.0), (900, 64, 0.0), (700, 100, 0.0),
                                       (1100, 128, 0.0)])
def test_dense_ragged_one_step(pkg, n, k, shift):
    p = synth.small_dense(n, k, m=8, seed=n + k, signs=True)
    p.shift = shift
    one_step(pkg, p, 3)


def test_cfg2_one_step_parity(pkg):
    p = synth.make_config("cfg2", device="cuda")
    worst, _ = one_step(pkg, p, 3)
    print(f"cfg2 worst {worst:.3e}")


def test_dense_intermediates(pkg):
    """P3: W, alpha, d, sigma, U, L=Y_1, T, E_11 and the materialised Y vs the oracle."""
    p = synth.small_dense(700, 24, m=8, seed=5, signs=True)
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    xin = X.clone()
    s, _ = R.refine_sweep(X, stats=True)
    assert s == pkg.REFINE_OK
    ref = oracle.sweep(op_of(p), xin.cpu().numpy(), debug=True)
    D = ref.debug
    sig = D["sigma"]
    A = p.A.numpy()
    Xn = xin.cpu().numpy()
    Wg = R.debug(pkg.DBG_W).cpu().numpy()           # un-flipped A X
    bound = 2 * p.n * U * (np.abs(A) @ np.abs(Xn))
    assert np.all(np.abs(Wg * sig - D["W"]) <= bound)
    assert np.array_equal(R.debug(pkg.DBG_SIGMA).cpu().numpy(), sig)
    assert rel(R.debug(pkg.DBG_ALPHA).cpu().numpy(), D["alpha"]) <= 1e-15
    assert rel(R.debug(pkg.DBG_D).cpu().numpy(), D["dtilde"]) <= 1e-14
    assert rel(R.debug(pkg.DBG_U).cpu().numpy(), D["U"]) <= 1e-13
    assert rel(R.debug(pkg.DBG_L).cpu().numpy(), D["Y"][:p.k]) <= 1e-13
    assert rel(R.debug(pkg.DBG_T).cpu().numpy(), D["T"]) <= 1e-13
    # E_11 = V_1/(d_j - d_i): rounding amplified by 1/gap; it enters X~ additively (|X| ~ 1)
    assert np.max(np.abs(R.debug(pkg.DBG_E11).cpu().numpy() - D["E"][:p.k])) <= 1e-12
    Y = R.debug(pkg.DBG_Y, xin).cpu().numpy()
    assert rel(Y, D["Y"]) <= 1e-13


def test_sign_flip_invariance_bitwise(pkg):
    p = synth.small_dense(600, 8, seed=3, signs=True)
    R = refiner(pkg, p)
    X1 = p.X0.cuda().clone()
    S = torch.tensor([1, -1, 1, -1, -1, 1, 1, -1], dtype=torch.float64, device="cuda")
    X2 = X1 * S
    R.refine_sweep(X1)
    R.refine_sweep(X2)
    assert torch.equal(X1, X2)


def test_deterministic_and_graph_mode(pkg):
    p = synth.small_dense(900, 16, seed=9)
    R = refiner(pkg, p)
    Xa, Xb, Xc = (p.X0.cuda().clone() for _ in range(3))
    R.refine_sweep(Xa)
    R.refine_sweep(Xb)
    assert torch.equal(Xa, Xb)
    R.refine_set_graph(True)
    R.refine_sweep(Xc)
    R.refine_sweep(Xc)           # replay
    R.refine_set_graph(False)
    R.refine_sweep(Xa)
    assert torch.equal(Xa, Xc)


def test_host_entry_point_matches_device(pkg):
    p = synth.small_dense(400, 6, seed=4)
    R = refiner(pkg, p)
    Xd = p.X0.cuda().clone()
    R.refine_sweep(Xd)
    Xh = p.X0.numpy().copy()
    s, st = R.refine_sweep_host(Xh)
    assert s == pkg.REFINE_OK
    assert np.array_equal(Xh, Xd.cpu().numpy())


@pytest.mark.parametrize("n,k", [(4096, 64), (6000, 32), (8192, 64)])
def test_host_entry_overlapped_upload(pkg, monkeypatch, n, k):
    """refine_sweep_host with the chunked upload overlapped with S1 (dense, TMA GEMM, >= 1 MiB of X^:
    the GEMM's producer waits per K step for its chunk's flag, the fix-up for its rows): bit-identical to
    the device sweep and to the plain upload, over several calls (the flags' epoch advances per call)."""
    p = synth.small_dense(n, k, m=8, seed=n + k, signs=True)
    R = refiner(pkg, p)
    Xd = p.X0.cuda().clone()
    Xh = p.X0.numpy().copy()
    for _ in range(3):
        R.refine_sweep(Xd)
        s, st = R.refine_sweep_host(Xh)
        assert s == pkg.REFINE_OK
        assert np.array_equal(Xh, Xd.cpu().numpy())
    Xpin = p.X0.clone().pin_memory()                 # pinned: the chunk copies are truly asynchronous
    R3 = refiner(pkg, p)
    for _ in range(3):
        s, st = R3.refine_sweep_host(Xpin)
        assert s == pkg.REFINE_OK
    assert np.array_equal(Xpin.numpy(), Xh)
    monkeypatch.setenv("REFINE_H2D_OVERLAP", "0")
    R2 = refiner(pkg, p)
    Xp = p.X0.numpy().copy()
    for _ in range(3):
        R2.refine_sweep_host(Xp)
    assert np.array_equal(Xp, Xh)


# ------------------------------------------------------------------------------ CSR

@pytest.mark.parametrize("dims,coeffs,k", [((40, 37), (1.0, 1.37), 6), ((64, 61), (1.0, 1.37), 32),
                                           ((17, 15, 13), (1.0, 1.13, 1.29), 20),
                                           ((24, 22, 21), (1.0, 1.13, 1.29), 128)])
def test_csr_one_step_and_bitwise_W(pkg, dims, coeffs, k):
    p = synth.small_laplacian(dims, coeffs, k)
    R = refiner(pkg, p)
    op = op_of(p)
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, _ = R.refine_sweep(X, stats=True)
    assert s == pkg.REFINE_OK
    ref = oracle.sweep(op, xin, debug=True)
    assert rel(X.cpu().numpy(), ref.X) <= TOL
    Wg = R.debug(pkg.DBG_W).cpu().numpy()
    assert np.array_equal(Wg * ref.debug["sigma"], ref.debug["W"])      # P3: bit-identical fma chains
    one_step(pkg, p, 3, R=R, op=op)


def test_csr_shift(pkg):
    """Sec. 5.1: L with shift = sigma (B = L - sigma I = -A') on the GPU vs the oracle."""
    p = synth.small_laplacian((30, 29), (1.0, 1.37), 5)
    rp, ci, v = p.row_ptr.numpy(), p.col_idx.numpy(), p.val.numpy()
    diag = ci == np.repeat(np.arange(p.n), np.diff(rp))
    p.val = torch.from_numpy(np.where(diag, p.meta["sigma"] - v, -v))
    p.shift = p.meta["sigma"]
    one_step(pkg, p, 2)


# ------------------------------------------------------------------------------ statuses

def test_near_zero_rq_leaves_X_unchanged(pkg):
    A = torch.diag(torch.tensor([0.0, 1.0, 2.0, 3.0] + [0.1] * 60, dtype=torch.float64)).cuda()
    R = pkg.Refiner.dense(A, 2)
    X = torch.zeros(64, 2, dtype=torch.float64, device="cuda")
    X[0, 0] = X[1, 1] = 1.0
    X0 = X.clone()
    s, _ = R.refine_sweep(X, stats=True)
    assert s == pkg.REFINE_E_NEAR_ZERO_RQ
    assert torch.equal(X, X0)


def test_nan_diverged(pkg):
    p = synth.small_dense(300, 4, seed=2)
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    X[17, 2] = float("nan")
    s, _ = R.refine_sweep(X, stats=True)
    assert s == pkg.REFINE_DIVERGED


def test_run_statuses(pkg):
    p = synth.make_config("cfg1")
    R = refiner(pkg, p)
    X = p.X0.cuda().clone()
    s, it, st = R.refine_run(X, 2, 1e-30)
    assert s == pkg.REFINE_MAXITER and it == 2
    s, it, st = R.refine_run(X, 50, 1e-12)
    assert s == pkg.REFINE_OK and st.corr_norm <= 1e-12 and it < 50
    Xo, so, ito, _ = oracle.run(op_of(p), p.X0.numpy(), 50, 1e-12)
    assert so == oracle.OK


# ------------------------------------------------------------------------------ row partition (loopback)

@pytest.mark.parametrize("world", [2, 3, 4])
def test_loopback_dense_row_partition(pkg, world):
    """The multi-rank code path (partitioned S1, gathered alpha/g, rank-0 k x k stage, broadcast,
    gathered norms) emulated on one device: one-step parity with the oracle and agreement with
    the single-rank run."""
    p = synth.small_dense(1003, 16, m=8, seed=17, signs=True)
    R = pkg.Refiner.dense(p.A.cuda(), p.k, world=world)
    one_step(pkg, p, 3, R=R)
    X1, Xp = p.X0.cuda().clone(), p.X0.cuda().clone()
    refiner(pkg, p).refine_sweep(X1)
    R.refine_sweep(Xp)
    assert rel(Xp.cpu().numpy(), X1.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("dims,k,world", [((40, 37), 6, 2), ((64, 8), 6, 16), ((17, 15, 13), 20, 3),
                                          ((24, 22, 21), 128, 4)])
def test_loopback_csr_halo(pkg, dims, k, world):
    """CSR row partition with halo exchange (incl. halos spanning several ranks at world=16)."""
    coeffs = (1.0, 1.37) if len(dims) == 2 else (1.0, 1.13, 1.29)
    p = synth.small_laplacian(dims, coeffs, k)
    R = pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, world=world)
    one_step(pkg, p, 2, R=R)
    X1, Xp = p.X0.cuda().clone(), p.X0.cuda().clone()
    refiner(pkg, p).refine_sweep(X1)
    R.refine_sweep(Xp)
    assert rel(Xp.cpu().numpy(), X1.cpu().numpy()) <= 1e-13


def test_loopback_run_converges(pkg):
    p = synth.make_config("cfg1")
    R = pkg.Refiner.dense(p.A.cuda(), p.k, world=2)
    X = p.X0.cuda().clone()
    s, it, st = R.refine_run(X, 40, 1e-14)
    assert s == pkg.REFINE_OK
    Xt = p.X.numpy()
    Xg = X.cpu().numpy()
    sg = np.sign(np.sum(Xg * Xt, axis=0))
    assert np.linalg.norm(Xg * sg - Xt, axis=0).max() <= 100 * p.n * U


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_nccl_path_single_rank(pkg, kind, monkeypatch):
    """The NCCL code path (all-gathers, broadcast, group send/recv) on a 1-rank communicator:
    REFINE_FORCE_NCCL=1 makes world == 1 take it.  One-step parity with the oracle."""
    monkeypatch.setenv("REFINE_FORCE_NCCL", "1")
    try:
        nid = pkg.refine_nccl_id()
    except pkg.RefineError:
        pytest.skip("NCCL not loadable")
    if kind == "dense":
        p = synth.small_dense(777, 12, m=8, seed=23, signs=True)
        R = pkg.Refiner.dense(p.A.cuda(), p.k, world=1, rank=0, nccl_id=nid)
    else:
        p = synth.small_laplacian((30, 21), (1.0, 1.37), 8)
        R = pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, world=1, rank=0, nccl_id=nid)
    assert R.kernels_per_sweep() in ((8, 9) if kind == "dense" else (8,))   # + kxk_lu, ag_local (dense: w_finish fused or not)
    one_step(pkg, p, 2, R=R)


def test_repeat_bitwise_k128(pkg):
    """Run-to-run determinism at the largest k (guards against races between CTAs)."""
    p = synth.small_dense(1100, 128, m=8, seed=1228, signs=True)
    R = refiner(pkg, p)
    outs = []
    for _ in range(4):
        X = p.X0.cuda().clone()
        R.refine_sweep(X)
        outs.append(X.cpu().numpy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


# ------------------------------------------------------------------------------ CSR gather kernel

@pytest.mark.parametrize("k", [2, 4, 8, 16, 64])
def test_csr_gather_every_k(pkg, k, monkeypatch):
    """spmm_gather_kernel instantiations (k a power of two): bit-identical W, one-step parity.
    (REFINE_SPMM=gather: 2-D grids with k a multiple of 32 take the stencil kernel by default.)"""
    monkeypatch.setenv("REFINE_SPMM", "gather")
    p = synth.small_laplacian((41, 37), (1.0, 1.37), k)
    R = refiner(pkg, p)
    op = op_of(p)
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    assert R.refine_sweep(X) == pkg.REFINE_OK
    ref = oracle.sweep(op, xin, debug=True)
    assert rel(X.cpu().numpy(), ref.X) <= TOL
    assert np.array_equal(R.debug(pkg.DBG_W).cpu().numpy() * ref.debug["sigma"], ref.debug["W"])


def _arrow(p, width, eps=1e-3):
    """Laplacian plus a symmetric 'arrow' coupling row/column 0 to columns 1..width-1 (long rows)."""
    import scipy.sparse as sp
    A = sp.csr_matrix((p.val.numpy(), p.col_idx.numpy(), p.row_ptr.numpy()), shape=(p.n, p.n))
    B = sp.lil_matrix((p.n, p.n))
    for j in range(1, width):
        B[0, j] = B[j, 0] = eps * (1.0 + (j % 7) / 7.0)
    C = (A + B.tocsr()).tocsr()
    C.sort_indices()
    import dataclasses
    return dataclasses.replace(p, row_ptr=torch.from_numpy(C.indptr.astype(np.int32)),
                               col_idx=torch.from_numpy(C.indices.astype(np.int32)),
                               val=torch.from_numpy(C.data.astype(np.float64)))


@pytest.mark.parametrize("width,k", [(700, 32), (3000, 32), (300, 128)])
def test_csr_gather_long_rows(pkg, width, k):
    """Rows with many nonzeros shrink the rows-per-chunk R (or fall back to the vec kernel when one
    chunk cannot be staged at all); the fma chains stay bit-identical to the oracle's."""
    q = _arrow(synth.small_laplacian((64, 61), (1.0, 1.37), k), width)
    R = refiner(pkg, q)
    op = op_of(q)
    X = q.X0.cuda().clone()
    xin = X.cpu().numpy()
    assert R.refine_sweep(X) == pkg.REFINE_OK
    ref = oracle.sweep(op, xin, debug=True)
    assert rel(X.cpu().numpy(), ref.X) <= TOL
    assert np.array_equal(R.debug(pkg.DBG_W).cpu().numpy() * ref.debug["sigma"], ref.debug["W"])


def test_csr_gather_matches_vec_kernel(pkg, monkeypatch):
    """The gather kernel and the previous vec kernel (REFINE_NO_GATHER=1) produce identical W
    (same fma chains); X agrees to rounding of the alpha / g partial-sum order."""
    p = synth.small_laplacian((24, 22, 21), (1.0, 1.13, 1.29), 64)
    Xa, Xb = p.X0.cuda().clone(), p.X0.cuda().clone()
    Ra = refiner(pkg, p)
    Ra.refine_sweep(Xa)
    monkeypatch.setenv("REFINE_NO_GATHER", "1")
    Rb = refiner(pkg, p)
    Rb.refine_sweep(Xb)
    assert torch.equal(Ra.debug(pkg.DBG_W), Rb.debug(pkg.DBG_W))
    assert rel(Xa.cpu().numpy(), Xb.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("dims,k", [((24, 22, 21), 128), ((24, 22, 21), 32), ((16, 15, 13), 8)])
def test_csr_stencil_chunk_order(pkg, dims, k, monkeypatch):
    """The tiled chunk order of the gather kernel (3-D stencils, spmm_csr.cuh chunk_of), forced on
    small grids: W bit-identical to the oracle's fma chains and one-step parity."""
    monkeypatch.setenv("REFINE_SPMM_ORDER", "1")
    p = synth.small_laplacian(dims, (1.0, 1.13, 1.29), k)
    R = refiner(pkg, p)
    op = op_of(p)
    X = p.X0.cuda().clone()
    xin = X.cpu().numpy()
    s, _ = R.refine_sweep(X, stats=True)
    assert s == pkg.REFINE_OK
    ref = oracle.sweep(op, xin, debug=True)
    assert rel(X.cpu().numpy(), ref.X) <= TOL
    assert np.array_equal(R.debug(pkg.DBG_W).cpu().numpy() * ref.debug["sigma"], ref.debug["W"])


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_run_conditional_graph_equals_enqueued_loop(pkg, kind, monkeypatch):
    """refine_run as one CUDA graph with a conditional WHILE node (single rank) gives bit for bit the
    result, status and sweep count of the enqueue-every-sweep loop (REFINE_RUN_NO_GRAPH=1), both when
    it converges early and when it exhausts the budget; with the reorthogonalisation policy too."""
    if kind == "dense":
        p = synth.make_config("cfg1")
    else:
        p = synth.small_laplacian((40, 37), (1.0, 1.37), 8, noise=1e-5)
    res = {}
    for mode in ("graph", "loop"):
        if mode == "loop":
            monkeypatch.setenv("REFINE_RUN_NO_GRAPH", "1")
        for iters, tol, kw in ((60, 1e-12, {}), (3, 1e-30, {}), (8, 1e-30, {"reorth_tol": 1e-30})):
            R = refiner(pkg, p, **kw)
            X = p.X0.cuda().clone()
            s, it, st = R.refine_run(X, iters, tol)
            res[(mode, iters, tol, tuple(kw))] = (s, it, st.corr_norm, X.cpu().numpy())
    for key, (s, it, c, X) in res.items():
        if key[0] != "graph":
            continue
        s2, it2, c2, X2 = res[("loop",) + key[1:]]
        assert (s, it) == (s2, it2), (key, s, it, s2, it2)
        assert c == c2 and np.array_equal(X, X2), key
    if kind == "dense":      # cfg1 converges in ~8 sweeps: the while loop stopped there
        assert res[("graph", 60, 1e-12, ())][0] == pkg.REFINE_OK and res[("graph", 60, 1e-12, ())][1] < 60


@pytest.mark.parametrize("kind,world", [("dense", 2), ("dense", 3), ("csr", 2), ("csr", 4)])
def test_graph_replay_row_partition(pkg, kind, world):
    """refine_set_graph at world > 1: the loopback ranks' kernels and collective copies are captured into
    one graph; replay equals direct launches bit for bit."""
    if kind == "dense":
        p = synth.small_dense(1003, 16, m=8, seed=17, signs=True)
        mk = lambda: pkg.Refiner.dense(p.A.cuda(), p.k, world=world)
    else:
        p = synth.small_laplacian((24, 22, 21), (1.0, 1.13, 1.29), 32)
        mk = lambda: pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, world=world)
    Ra, Rb = mk(), mk()
    Xa, Xb = p.X0.cuda().clone(), p.X0.cuda().clone()
    Rb.refine_set_graph(True)
    for _ in range(3):
        Ra.refine_sweep(Xa)
        Rb.refine_sweep(Xb)
    assert torch.equal(Xa, Xb)


@pytest.mark.parametrize("kind", ["dense", "csr"])
def test_nccl_path_single_rank_graph(pkg, kind, monkeypatch):
    """The NCCL calls (group broadcast / send-recv, all-gathers, broadcast) captured in the sweep's CUDA
    graph on a 1-rank communicator (REFINE_FORCE_NCCL=1): replay equals direct launches."""
    monkeypatch.setenv("REFINE_FORCE_NCCL", "1")
    try:
        nid = pkg.refine_nccl_id()
    except pkg.RefineError:
        pytest.skip("NCCL not loadable")
    if kind == "dense":
        p = synth.small_dense(777, 12, m=8, seed=23, signs=True)
        mk = lambda i: pkg.Refiner.dense(p.A.cuda(), p.k, world=1, rank=0, nccl_id=i)
    else:
        p = synth.small_laplacian((30, 21), (1.0, 1.37), 8)
        mk = lambda i: pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, world=1, rank=0,
                                       nccl_id=i)
    Ra = mk(nid)
    Rb = mk(pkg.refine_nccl_id())
    Xa, Xb = p.X0.cuda().clone(), p.X0.cuda().clone()
    Rb.refine_set_graph(True)
    for _ in range(3):
        Ra.refine_sweep(Xa)
        Rb.refine_sweep(Xb)
    assert torch.equal(Xa, Xb)


# ------------------------------------------------------------------------------ k x k chain variants

@pytest.mark.parametrize("env", [{}, {"REFINE_KXK_CL16": "0"}, {"REFINE_FK_BULK": "0"},
                                 {"REFINE_KXK_H": "0"}, {"REFINE_KXK_CL16": "0", "REFINE_KXK_H": "0"}],
                         ids=["cl16-bulk-H", "cl8", "cp.async", "no-H", "cl8-no-H"])
@pytest.mark.parametrize("k", [96, 128])
def test_kxk_finish_variants(pkg, monkeypatch, env, k):
    """kxk_finish's clustered paths at k > 64 (kxk.cuh): the 16-CTA cluster (8-row blocks, per-CTA
    statistics slots) and the 8-CTA fallback, bulk-copy and cp.async staging of the products, the
    paired H products and the three-stage T form -- each one-step parity with the oracle, per row block
    and column (k = 96: ragged cluster rows, some CTAs without rows)."""
    for kk, v in env.items():
        monkeypatch.setenv(kk, v)
    p = synth.small_dense(1200, k, m=8, seed=7 + k, signs=True)
    worst, _ = one_step(pkg, p, 2)
    print(f"k={k} {env}: worst one-step rel diff {worst:.3e}")


def test_passC_pp_variants_bitwise(pkg, monkeypatch):
    """The k = 128 ping-pong pass C in its three ring shapes (passes.cuh PassCPPCfgT: 2 stages of 32 rows,
    3 of 24 (default), 4 of 16): every output element has the same DMMA k-order and epilogue fma, so the
    sweeps agree bit for bit; one-step parity with the oracle on the default."""
    p = synth.small_dense(1500, 128, m=8, seed=1628, signs=True)
    outs = []
    for v in ("1", "3", "4"):
        monkeypatch.setenv("REFINE_PASSC_PP", v)
        R = refiner(pkg, p)
        X = p.X0.cuda().clone()
        for _ in range(2):
            assert R.refine_sweep(X) == pkg.REFINE_OK
        outs.append(X.cpu().numpy())
        del R
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    monkeypatch.setenv("REFINE_PASSC_PP", "3")
    worst, _ = one_step(pkg, p, 2)
    print(f"pass C variants: worst one-step rel diff {worst:.3e}")
