import sys, torch, numpy as np
sys.path.insert(0, ".")
import synth, paper_2602_23778_b200 as pkg
mixed = bool(int(sys.argv[1])); k = int(sys.argv[2]); kind = sys.argv[3]
if kind == "dense":
    p = synth.small_dense(1100, k, m=8, noise=1e-5, seed=7, signs=True)
    R = pkg.Refiner.dense(p.A.cuda(), p.k, shift=p.shift, mixed=mixed)
else:
    p = synth.small_laplacian((24, 22, 21), (1.0, 1.13, 1.29), k, noise=1e-5)
    R = pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k, shift=p.shift, mixed=mixed)
buf = torch.empty(p.n * p.k + 1, dtype=torch.float64, device="cuda")
X = buf[1:].view(p.n, p.k)
X.copy_(p.X0.cuda())
s, st = R.refine_sweep(X, stats=True)
print("mixed", mixed, "k", k, kind, "status", s)
