"""Small workload touching every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, one tool per run):  compute-sanitizer --tool X python tools/sanitize_run.py
Dense: cfg1 (k = 4), k = 16 / 32 (one-CTA k x k), k = 64 / 128 (clustered kxk_finish, pass B2), the
tcgen05 passes (mixed), the INT8 Ozaki S1 / pass C (emul); CSR: gather SpMM (2-D) and the TMA
stencil SpMM (3-D), Rayleigh-Ritz, reorthogonalisation, refine_run with graph replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_23778_b200 as pkg  # noqa: E402
import synth  # noqa: E402


def run(R, X0, sweeps=2, rr=False):
    X = X0.cuda().clone()
    for _ in range(sweeps):
        s, st = R.refine_sweep(X, stats=True)
        assert s == pkg.REFINE_OK, s
    if rr:
        assert R.refine_rayleigh_ritz(X)[0] == pkg.REFINE_OK
        assert R.refine_reorthogonalize(X)[0] == pkg.REFINE_OK
    torch.cuda.synchronize()


cases = []
p = synth.make_config("cfg1")
cases.append(("cfg1", lambda: pkg.Refiner.dense(p.A.cuda(), p.k), p, True))
for n, k in ((700, 16), (900, 32), (1000, 64), (1100, 128)):
    q = synth.small_dense(n, k, m=8, seed=n, signs=True)
    cases.append((f"dense {n}x{k}", (lambda q=q: pkg.Refiner.dense(q.A.cuda(), q.k)), q, k == 64))
q = synth.small_dense(1024, 64, m=8, seed=4)
cases.append(("mixed 1024x64", lambda q=q: pkg.Refiner.dense(q.A.cuda(), q.k, mixed=2), q, False))
cases.append(("emul 1024x64", lambda q=q: pkg.Refiner.dense(q.A.cuda(), q.k, emul=True), q, False))
c2 = synth.small_laplacian((64, 61), (1.0, 1.37), 32)
cases.append(("csr2d k32 gather", lambda: pkg.Refiner.csr(c2.row_ptr.cuda(), c2.col_idx.cuda(), c2.val.cuda(), c2.n, c2.k), c2, True))
c3 = synth.small_laplacian((24, 22, 21), (1.0, 1.13, 1.29), 128)
cases.append(("csr3d k128 stencil", lambda: pkg.Refiner.csr(c3.row_ptr.cuda(), c3.col_idx.cuda(), c3.val.cuda(), c3.n, c3.k), c3, False))
cases.append(("csr3d k128 emul", lambda: pkg.Refiner.csr(c3.row_ptr.cuda(), c3.col_idx.cuda(), c3.val.cuda(), c3.n, c3.k, emul=True), c3, False))
for name, make, prob, rr in cases:
    R = make()
    run(R, prob.X0, rr=rr)
    print("ok", name, flush=True)
    del R
R = pkg.Refiner.dense(p.A.cuda(), p.k)
R.refine_set_graph(True)
X = p.X0.cuda().clone()
R.refine_sweep(X)
R.refine_sweep(X)
R.refine_set_graph(False)
s, it, st = R.refine_run(X, 5, 1e-30)
torch.cuda.synchronize()
print("ok graph + refine_run", s, it, flush=True)
