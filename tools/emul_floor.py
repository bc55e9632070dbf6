"""Convergence floor of the INT8-emulated S1 vs DMMA: corr_norm / rel_resid after many sweeps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2602_23778_b200 as pkg
for seed, n, k in ((29, 3000, 64), (5, 2000, 32), (7, 4096, 16)):
    p = synth.small_dense(n, k, m=8, noise=1e-6, seed=seed)
    for emul in (False, True):
        R = pkg.Refiner.dense(p.A.cuda(), k, emul=emul)
        X = p.X0.cuda().clone()
        cs = []
        for t in range(25):
            s, st = R.refine_sweep(X, stats=True)
            cs.append(st.corr_norm)
        Xg, Xt = X.cpu().numpy(), p.X.numpy()
        sg = np.sign(np.sum(Xg * Xt, axis=0))
        err = np.linalg.norm(Xg * sg - Xt, axis=0).max()
        print(f"n={n} k={k} emul={emul}: corr {min(cs[-10:]):.2e}..{max(cs[-10:]):.2e} resid {st.rel_resid:.2e} "
              f"err {err:.2e} (100nu {100 * n * 2**-53:.2e})")
