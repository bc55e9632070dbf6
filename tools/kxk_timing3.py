"""kxk_finish device time (per-kernel CUDA events of refine_profile_begin/end) at k = 4 .. 128."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2602_23778_b200 as pkg
for (n, k) in [(256, 4), (4096, 16), (8192, 32), (8192, 64), (8192, 128)]:
    p = synth.small_dense(n, k, m=8, seed=3, signs=True, device="cuda")
    R = pkg.Refiner.dense(p.A, k)
    X = p.X0.clone()
    for _ in range(3):
        R.refine_sweep(X)
    R.refine_profile_begin(10)
    for _ in range(10):
        R.refine_sweep(X)
    kern, ns = R.refine_profile_end()
    print(f"k={k}: " + "  ".join(f"{a} {1000 * v / ns:.1f}us" for a, v in kern.items()))
