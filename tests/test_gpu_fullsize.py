"""Full-size parity at BASELINE.json's configs, in the launch configuration bench.py times
(same library defaults): one-step parity P1 -- the oracle (on the host cores) consumes
the GPU's own input X_t and the GPU's X_{t+1} must match within relative Frobenius 1e-10
(north_star).  For the CSR configs W is also checked bit-identical (P3).  Each config runs
its first sweep (the largest correction, eps_0 ~ 1e-6..1e-3) and one later sweep."""
import time

import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import compare_sweep

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def pkg():
    import paper_2602_23778_b200 as p
    from paper_2602_23778_b200 import build
    build.build()
    p.lib()
    return p


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_fullsize_one_step(pkg, name):
    p = synth.make_config(name, device="cuda")
    if p.kind == "dense":
        R = pkg.Refiner.dense(p.A, p.k, shift=p.shift)
        op = oracle.Operator(A=p.A.cpu().numpy(), shift=p.shift)
    else:
        R = pkg.Refiner.csr(p.row_ptr, p.col_idx, p.val, p.n, p.k, shift=p.shift)
        op = oracle.Operator(row_ptr=p.row_ptr.cpu().numpy(), col_idx=p.col_idx.cpu().numpy(),
                             val=p.val.cpu().numpy(), shift=p.shift)
    normA = op.norm_inf()
    X = p.X0.clone()
    for t in range(2):
        if t == 1:           # advance a few sweeps on the GPU, then check one more
            for _ in range(2):
                R.refine_sweep(X)
        xin = X.cpu().numpy()
        s, st = R.refine_sweep(X, stats=True)
        assert s == pkg.REFINE_OK
        t0 = time.perf_counter()
        ref = oracle.sweep(op, xin, debug=True)
        dt = time.perf_counter() - t0
        assert ref.status == oracle.OK
        sig = ref.debug["sigma"]
        e = compare_sweep(X.cpu().numpy(), ref, st, k=p.k, where=f"{name} t={t}", normA=normA)
        print(f"{name} t={t} one-step rel {e:.3e} (oracle {dt:.1f}s, {oracle.num_threads()} threads) "
              f"corr gpu {st.corr_norm:.6e} oracle {ref.stats.corr_norm:.6e} min_gap {st.min_gap:.3e}")
        if p.kind == "csr":
            Wg = R.debug(pkg.DBG_W).cpu().numpy()
            assert np.array_equal(Wg * sig, ref.debug["W"])
        del ref
