"""A few sweeps of one config with refine_opts.emul (or mixed) for ncu captures of oz_gemm /
passC_oz (passB_tc / passC_tc).
  python tools/emul_run.py cfg3 [sweeps] [emul|mixed]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2602_23778_b200 as pkg
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
opt = {"emul": True} if (sys.argv[3] if len(sys.argv) > 3 else "emul") == "emul" else {"mixed": 1}
p = synth.make_config(name, device="cuda")
R = (pkg.Refiner.dense(p.A, p.k, **opt) if p.kind == "dense" else
     pkg.Refiner.csr(p.row_ptr, p.col_idx, p.val, p.n, p.k, **opt))
X = p.X0.clone()
for _ in range(sweeps):
    s, st = R.refine_sweep(X, stats=True)
torch.cuda.synchronize()
print(name, "status", s, "rel_resid", st.rel_resid)
