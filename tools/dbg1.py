import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, synth, paper_2602_23778_b200 as pkg
p = synth.small_dense(1100, 128, m=8, seed=1228, signs=True)
R = pkg.Refiner.dense(p.A.cuda(), p.k)
op = oracle.Operator(A=p.A.numpy())
X = p.X0.cuda().clone()
for t in range(4):
    xin = X.cpu().numpy()
    s, st = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(op, xin, debug=True)
    Xg = X.cpu().numpy()
    sig = ref.debug['sigma']
    cg = Xg - xin*sig; co = ref.X - xin*sig
    print(t, 'relX %.2e' % (np.linalg.norm(Xg-ref.X)/np.linalg.norm(ref.X)), 'relcorr %.2e' % (np.linalg.norm(cg-co)/np.linalg.norm(co)),
          'corr g %.6e o %.6e rel %.2e' % (st.corr_norm, ref.stats.corr_norm, abs(st.corr_norm-ref.stats.corr_norm)/ref.stats.corr_norm),
          'rr %.3e %.3e' % (st.rel_resid, ref.stats.rel_resid), 'E11 %.3e' % np.linalg.norm(ref.debug['E'][:128]), 'E2 %.3e' % np.linalg.norm(ref.debug['E'][128:]))
