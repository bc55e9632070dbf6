import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, synth, paper_2602_23778_b200 as pkg
p = synth.small_dense(1100, 128, m=8, seed=1228, signs=True)
R = pkg.Refiner.dense(p.A.cuda(), p.k)
outs = []
for rep in range(6):
    X = p.X0.cuda().clone()
    R.refine_sweep(X)
    outs.append(X.cpu().numpy())
print('bitwise repeat:', [bool(np.array_equal(outs[0], o)) for o in outs[1:]], [float(np.abs(outs[0]-o).max()) for o in outs[1:]])
for kk in [64, 100, 128]:
    q = synth.small_dense(900, kk, m=8, seed=5, signs=True)
    Rq = pkg.Refiner.dense(q.A.cuda(), q.k)
    o = []
    for rep in range(6):
        X = q.X0.cuda().clone(); Rq.refine_sweep(X); o.append(X.cpu().numpy())
    print(kk, 'repeat max diff', max(float(np.abs(o[0]-x).max()) for x in o[1:]))
