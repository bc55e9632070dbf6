"""Repeat one sweep from the same input many times; for every output that differs bitwise from the
first, report where: W (S1), d (S2), and the top / lower rows of X (kxk_finish / pass C)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_23778_b200 as pkg  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
p = synth.make_config(name, device="cuda")
R = pkg.Refiner.dense(p.A, p.k)
X = p.X0.clone()
for _ in range(3):
    R.refine_sweep(X)
xin = X.clone()
first = None
nbad = 0
for rep in range(reps):
    Y = xin.clone()
    R.refine_sweep(Y)
    W = R.debug(pkg.DBG_W).cpu().numpy()
    d = R.debug(pkg.DBG_D).cpu().numpy()
    E = R.debug(pkg.DBG_E11).cpu().numpy()
    T = R.debug(pkg.DBG_T).cpu().numpy()
    Yh = Y.cpu().numpy()
    cur = (W, d, E, T, Yh)
    if first is None:
        first = cur
        continue
    if not np.array_equal(Yh, first[4]):
        nbad += 1
        dW = np.abs(W - first[0]); rows = np.unique(np.nonzero(dW)[0])
        print(f"rep {rep}: W diff max {dW.max():.3e} in {len(rows)} rows {rows[:8]}..., d diff {np.abs(d - first[1]).max():.3e}, "
              f"E11 diff {np.abs(E - first[2]).max():.3e}, T diff {np.abs(T - first[3]).max():.3e}, "
              f"X top {np.abs(Yh[:p.k] - first[4][:p.k]).max():.3e} lower {np.abs(Yh[p.k:] - first[4][p.k:]).max():.3e}",
              flush=True)
print(f"{name}: {nbad} of {reps - 1} repeats differ", flush=True)
