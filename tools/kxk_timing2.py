import os, sys
os.environ["REFINE_KXK_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2602_23778_b200 as pkg
for (n, k) in [(256, 4), (4096, 16), (8192, 64), (8192, 128)]:
    p = synth.small_dense(n, k, m=8, seed=3, signs=True, device="cuda")
    R = pkg.Refiner.dense(p.A, k)
    X = p.X0.clone()
    for _ in range(3):
        t = torch.zeros(64, dtype=torch.float64, device="cuda")
        R.refine_sweep(X, stats=True)
    R.refine_debug_get(10, t)
    v = t.cpu().numpy().view(np.int64)
    g = v[40:40 + int(v[55])] if 0 < v[55] < 16 else v[40:56]
    print(f"k={k}: first cta_gemm phases {np.diff(g).tolist()}")
