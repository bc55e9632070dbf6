"""Per-config sweep time with direct launches vs CUDA-graph replay (refine_set_graph)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2602_23778_b200 as pkg

for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "cfg3"]:
    p = bench.make_problem(name, "cuda:0")
    for graph in (False, True):
        R, X = bench.make_refiner(p, 1, 0)
        if graph:
            R.refine_set_graph(True)
        for _ in range(5):
            R.refine_sweep(X)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 50 if p.n < 100000 else 10
        e0.record()
        for _ in range(steps):
            R.refine_sweep(X)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} graph={graph}: {e0.elapsed_time(e1) / steps * 1000:.1f} us/sweep", flush=True)
        del R, X
    del p
    torch.cuda.empty_cache()
