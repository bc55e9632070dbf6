"""A few sweeps at n = 8192, k = 128 (dense): the kxk kernels for an ncu capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2602_23778_b200 as pkg
k = int(sys.argv[1]) if len(sys.argv) > 1 else 128
p = synth.small_dense(8192, k, m=8, seed=3, signs=True, device="cuda")
R = pkg.Refiner.dense(p.A, k)
X = p.X0.clone()
for _ in range(3):
    R.refine_sweep(X, stats=True)
torch.cuda.synchronize()
