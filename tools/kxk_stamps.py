"""kxk_finish phase stamps (clock64 on CTA 0 after each cluster barrier; REFINE_KXK_TIMING=1)."""
import os, sys
os.environ["REFINE_KXK_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_2602_23778_b200 as pkg
for (n, k) in [(256, 4), (4096, 16), (8192, 32), (8192, 64), (8192, 128)]:
    torch.cuda.synchronize()
    p = synth.small_dense(n, k, m=8, seed=3, signs=True, device="cuda")
    R = pkg.Refiner.dense(p.A, k)
    X = p.X0.clone()
    for _ in range(3):
        R.refine_sweep(X, stats=True)
    t = torch.zeros(64, dtype=torch.float64, device="cuda")
    R.refine_debug_get(10, t)
    a = t.cpu().numpy().view(np.int64)
    v = a[20:33]
    v = v[v != 0]
    print(f"k={k}: total {(v[-1] - v[0]) / 1.965e3:.1f} us  phases " + " ".join(f"{x / 1.965e3:.1f}" for x in np.diff(v)))
    if a[56] and a[59]:
        print(f"   first cta_gemm_fullk: staging {(a[57] - a[56]) / 1.965e3:.2f} us, DMMA+stores {(a[58] - a[57]) / 1.965e3:.2f} us, "
              f"final barrier {(a[59] - a[58]) / 1.965e3:.2f} us")
    if a[60] and a[63]:
        print(f"   second cta_gemm_fullk: staging {(a[61] - a[60]) / 1.965e3:.2f} us, DMMA+stores {(a[62] - a[61]) / 1.965e3:.2f} us, "
              f"final barrier {(a[63] - a[62]) / 1.965e3:.2f} us")
    if a[35] and a[36]:
        print(f"   first phase: start -> elementwise {(a[35] - a[20]) / 1.965e3:.1f} us, elementwise {(a[36] - a[35]) / 1.965e3:.1f} us, "
              f"cluster barrier {(a[22] - a[36]) / 1.965e3:.1f} us")
    if a[33] and a[34]:
        print(f"   stats phase: column sums {(a[33] - a[30]) / 1.965e3:.1f} us, per-column {(a[34] - a[33]) / 1.965e3:.1f} us, "
              f"tail {(a[31] - a[34]) / 1.965e3:.1f} us")
