import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, synth, paper_2602_23778_b200 as pkg
def rel(a,b): return float(np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300))
for (n,k) in [(1100,100),(1100,128),(700,64)]:
    p = synth.small_dense(n, k, m=8, seed=n+k, signs=True)
    R = pkg.Refiner.dense(p.A.cuda(), p.k)
    X = p.X0.cuda().clone(); xin = X.clone()
    s, st = R.refine_sweep(X, stats=True)
    ref = oracle.sweep(oracle.Operator(A=p.A.numpy()), xin.cpu().numpy(), debug=True)
    D = ref.debug
    out = {'X': rel(X.cpu().numpy(), ref.X)}
    out['d'] = rel(R.debug(pkg.DBG_D).cpu().numpy(), D['dtilde'])
    out['sig'] = float(np.abs(R.debug(pkg.DBG_SIGMA).cpu().numpy()-D['sigma']).max())
    out['U'] = rel(R.debug(pkg.DBG_U).cpu().numpy(), D['U'])
    out['L'] = rel(R.debug(pkg.DBG_L).cpu().numpy(), D['Y'][:k])
    out['T'] = rel(R.debug(pkg.DBG_T).cpu().numpy(), D['T'])
    out['E11'] = float(np.abs(R.debug(pkg.DBG_E11).cpu().numpy()-D['E'][:k]).max())
    Wg = R.debug(pkg.DBG_W).cpu().numpy()*D['sigma']
    out['W'] = rel(Wg, D['W'])
    print(n,k,s,{a:f"{b:.2e}" for a,b in out.items()})
