"""refine_run wall time per iteration (device events) on small configs: graph-replayed iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2602_23778_b200 as pkg
for name in ("cfg1", "cfg2", "cfg4"):
    p = synth.make_config(name, device="cuda")
    R = (pkg.Refiner.dense(p.A, p.k) if p.kind == "dense" else
         pkg.Refiner.csr(p.row_ptr, p.col_idx, p.val, p.n, p.k))
    X = p.X0.clone()
    R.refine_run(X, 5, 0.0)                # warm (captures the graph)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    X = p.X0.clone()
    e0.record()
    s, it, st = R.refine_run(X, 20, 0.0)   # tol 0: every iteration runs
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: refine_run {e0.elapsed_time(e1) / 20 * 1000:.1f} us/iteration (status {s}, {it} iterations)")
