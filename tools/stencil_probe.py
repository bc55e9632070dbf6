import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["REFINE_VERBOSE"] = "1"
import synth, paper_2602_23778_b200 as pkg
for dims, co, k in [((64, 61), (1.0, 1.37), 32), ((24, 22, 21), (1.0, 1.13, 1.29), 128)]:
    p = synth.small_laplacian(dims, co, k)
    R = pkg.Refiner.csr(p.row_ptr.cuda(), p.col_idx.cuda(), p.val.cuda(), p.n, p.k)
    print(dims, k, R.debug(pkg.DBG_SPMM).cpu().numpy().tolist(), flush=True)
p = synth.make_config("cfg5", device="cuda")
R = pkg.Refiner.csr(p.row_ptr, p.col_idx, p.val, p.n, p.k)
print("cfg5", R.debug(pkg.DBG_SPMM).cpu().numpy().tolist(), flush=True)
