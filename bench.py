#!/usr/bin/env python
"""Benchmark of the refinement sweep (arXiv 2602.23778 Alg. 4) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

A "step" is one sweep (all SURVEY.md Sec. 8(a) steps) over the config's X^ (n x k).
Headline workload: BASELINE.json configs[2] (cfg3: dense FP64 n=32768, k=64) -- the
largest dense config, whose 8.6 GB A is larger than L2 (so no flush is needed between
timed sweeps).  Metric: sweeps/s (BASELINE.json "refinement sweeps/s per config").
Rank 0 prints ONE JSON line.  Other configs are reported under "per_config" (sweeps/s
and roofline fraction each, smaller K).

--impl reference times the oracle (oracle/, the plain CPU program the parity tests
trust) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
METRIC = "refinement sweeps/s"


def peaks():
    hbm = 6547.5
    try:
        hbm = json.load(open(PEAKS_FILE))["hbm_gbs"]
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        hbm_src = "fallback"
    fp64 = json.load(open(FP64_FILE))["dmma_fp64_tflops"]
    return hbm, hbm_src, fp64


def alg_counts(p):
    """Per-sweep algorithmic flops and bytes (Table 1, FMA = 2 flops)."""
    n, k = p.n, p.k
    if p.kind == "dense":
        f = 2.0 * n * n * k + 8.0 * n * k * k
        b = 8.0 * n * n + 16.0 * n * k
    else:
        f = 2.0 * p.nnz * k + 8.0 * n * k * k
        b = 12.0 * p.nnz + 4.0 * (n + 1) + 16.0 * n * k
    return f, b


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    elif args.impl != "reference":
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device="cuda"):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_problem(name, device):
    import synth
    return synth.make_config(name, device=device)


def partition(n, world, rank):
    """Row blocks of the multi-GPU path (rank 0 takes the remainder; it must own rows 0..k-1)."""
    blk = n // world
    rb = 0 if rank == 0 else n - blk * (world - rank)
    return rb, n - blk * (world - rank - 1)


def make_refiner(p, world, rank, **opts):
    """Refiner for this rank: world == 1 -> whole problem; world > 1 -> row partition over NCCL
    (ncclUniqueId from rank 0, broadcast over torch.distributed).  Returns (Refiner, X_local)."""
    import torch
    import paper_2602_23778_b200 as pkg
    stream = torch.cuda.current_stream()
    if world == 1:
        if p.kind == "dense":
            return pkg.Refiner.dense(p.A, p.k, shift=p.shift, stream=stream, **opts), p.X0.clone()
        return (pkg.Refiner.csr(p.row_ptr, p.col_idx, p.val, p.n, p.k, shift=p.shift, stream=stream, **opts),
                p.X0.clone())
    import torch.distributed as dist
    obj = [pkg.refine_nccl_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    rb, re = partition(p.n, world, rank)
    kw = dict(shift=p.shift, stream=stream, row_begin=rb, row_end=re, rank=rank, world=world, nccl_id=obj[0], **opts)
    if p.kind == "dense":
        R = pkg.Refiner.dense(p.A[rb:re], p.k, n=p.n, **kw)
    else:
        R = pkg.Refiner.csr(p.row_ptr[rb:re + 1].contiguous(), p.col_idx, p.val, p.n, p.k, **kw)
    return R, p.X0[rb:re].clone()


def time_ours(p, steps, warmup, world, local, profile=True, rank=0, opts=None):
    """Device-timed sweeps: CUDA events on the library's stream, barrier + sync on both sides.

    The timed value replays the sweep as a CUDA graph (refine_set_graph) with no instrumentation;
    a second, separately timed pass launches the kernels directly with per-kernel CUDA events
    (refine_profile_begin/end) for the kernel breakdown and the roofline of the dominant kernel."""
    import torch
    stream = torch.cuda.current_stream()
    R, X = make_refiner(p, world, rank, **(opts or {}))

    def timed(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(n):
            R.refine_sweep(X)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        return e0.elapsed_time(e1) / n

    R.refine_set_graph(True)        # (world > 1: the NCCL calls are captured with the kernels; replay
                                    #  parity-tested on a 1-rank communicator and loopback ranks)
    for _ in range(warmup):
        R.refine_sweep(X)
    torch.cuda.synchronize()
    ms = timed(steps)
    R.refine_set_graph(False)
    kern, ms_prof = None, None
    if profile:
        for _ in range(2):
            R.refine_sweep(X)
        R.refine_profile_begin(steps)
        ms_prof = timed(steps)
        kern, ns = R.refine_profile_end()
        kern = {k_: v / max(ns, 1) for k_, v in kern.items()}       # ms per launch
    s, st = R.refine_sweep(X, stats=True)
    return ms, kern, R, X, st, s, ms_prof


def time_rr(R, X, reps=3):
    """Rayleigh-Ritz preprocessing (NEXT-1, Sec. 3.4): device time of refine_rayleigh_ritz."""
    import torch
    X = X.clone()
    R.refine_rayleigh_ritz(X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        s, _ = R.refine_rayleigh_ritz(X)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, s


def time_mixed(q, local, steps=5):
    """NEXT-2 (opts.mixed, k a multiple of 16, >= 32): the same sweep with passes B and C on tcgen05 in the
    bf16x3 scheme; device-timed like the FP64 sweep (graph replay)."""
    import torch
    if q.k % 16 or q.k < 32:
        return None
    ms, kern, R, X, st, s, prof = time_ours(q, steps, 3, 1, local, opts={"mixed": True})
    out = {"sweeps_s": 1000.0 / ms, "ms_per_sweep": ms, "ms_per_sweep_instrumented": prof, "kernels_ms": kern,
           "status": s, "what": "refine_opts.mixed: X_2^T [R_2|X_2] and X_2 Csig on tcgen05 (bf16x3 split, FP32 "
           "TMEM accumulators drained to FP64 every 512 rows); R, w scaling, k x k and reductions FP64"}
    del R, X
    torch.cuda.empty_cache()
    return out


def time_emul(q, local, steps=5):
    """Dense S1 with FP64 accuracy on the INT8 tensor cores (refine_opts.emul, ozaki.cuh; k a
    multiple of 16, <= 64): the same sweep, device-timed (graph replay)."""
    import torch
    if not ((q.kind == "dense" and q.k % 16 == 0 and q.k <= 64) or q.k == 128):
        return None
    ms, kern, R, X, st, s, prof = time_ours(q, steps, 3, 1, local, opts={"emul": True})
    out = {"sweeps_s": 1000.0 / ms, "ms_per_sweep": ms, "ms_per_sweep_instrumented": prof, "kernels_ms": kern,
           "status": s, "what": "refine_opts.emul: dense k <= 64: W = A X^ from 7 balanced 8-bit int8 digits of A (rows, once) "
           "and X^ (columns, per sweep) on tcgen05.mma kind::i8 with exact int32 level sums combined in FP64 "
           "(diagonal in FP64; the gemm_ax slot includes the per-sweep X slicing); k = 128: pass C "
           "(X_2 Csig) on kind::i8 with 5 x 7-bit digits"}
    del R, X
    torch.cuda.empty_cache()
    return out


def time_e2e(R, p, steps, warmup, world=1, rank=0):
    """Host buffers through the C ABI: H2D of X^, sweep, D2H of the result, each step."""
    import torch
    rb, re = partition(p.n, world, rank)
    Xh = p.X0[rb:re].cpu().pin_memory()
    R.refine_set_graph(True)        # the sweep between the copies replays its CUDA graph, as in `value`
    for _ in range(max(1, warmup)):
        R.refine_sweep_host(Xh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        s, st = R.refine_sweep_host(Xh)
    t1 = time.perf_counter()
    R.refine_set_graph(False)
    nb = (re - rb) * p.k * 8
    return (t1 - t0) / steps, nb, nb + 40


def roofline_for(p, kern, ms_step, fp64_peak, hbm_peak, n_loc=None):
    """Dominant kernel: its algorithmic flops (bytes) per launch / its average launch time
    (per rank: n_loc local rows of the row partition)."""
    if not kern:
        return None
    top = max(kern, key=kern.get)
    n, k = p.n, p.k
    nl = n if n_loc is None else n_loc
    traffic = None
    try:
        tr = json.load(open(TRAFFIC_FILE))
        traffic = tr.get(p.name, {}).get(top)
    except Exception:
        pass
    t = kern[top] * 1e-3
    if top == "gemm_ax":
        flops = 2.0 * nl * n * k
        ach = flops / t / 1e12
        return {"kernel": top, "bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": ach / fp64_peak, "traffic": traffic, "share_of_step": kern[top] / ms_step,
                "per_launch_alg": f"2*n*n*k = {flops:.4g} flop (FP64 DMMA)",
                "peak_source": "DMMA FP64 microbenchmark on this pool's B200 (profiles/r01_fp64_peaks.json)"}
    if top in ("passB", "passC"):
        rows = nl - k
        fl = (4.0 if top == "passB" else 2.0) * rows * k * k
        by = (16.0 if top == "passB" else 24.0) * rows * k
        t_f, t_b = fl / (fp64_peak * 1e12), by / (hbm_peak * 1e9)
        if t_f >= t_b:
            ach = fl / t / 1e12
            r = {"kernel": top, "bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                 "frac": ach / fp64_peak, "traffic": traffic, "share_of_step": kern[top] / ms_step,
                 "per_launch_alg": f"{fl:.4g} flop", "peak_source": "DMMA FP64 microbenchmark"}
            if top == "passB" and k == 128:
                # Table 1 credits 4 n k^2 (M and G in full); passB2_pp_kernel issues M (2 n k^2) plus 20 of
                # G's 32 warp tiles of 32 x 16 (those on or above its diagonal): 3.25 n k^2 executed
                ex = 3.25 * rows * k * k
                r["frac_executed"] = ex / t / 1e12 / fp64_peak
                r["executed_flop"] = f"{ex:.4g} flop (M + the G warp tiles on / above the diagonal)"
            return r
        ach = by / t / 1e9
        return {"kernel": top, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "traffic": traffic, "share_of_step": kern[top] / ms_step,
                "per_launch_alg": f"{by:.4g} bytes", "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    if top == "spmm_csr":
        by = 12.0 * p.nnz + 4.0 * (n + 1) + 16.0 * n * k
        ach = by / t / 1e9
        return {"kernel": top, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "traffic": traffic, "share_of_step": kern[top] / ms_step,
                "per_launch_alg": f"A + X + W = {by:.4g} bytes", "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    return {"kernel": top, "bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
            "traffic": traffic, "share_of_step": kern[top] / ms_step}


def s1_roofline(p, kern):
    """S1 (W = A X^) of a CSR config against HBM: algorithmic bytes A (values + column indices + row
    pointers) + X^ read + W written, over the kernel's CUDA-event time (north_star: >= 70 %)."""
    if p.kind != "csr" or "spmm_csr" not in kern:
        return None
    hbm, src, _ = peaks()
    by = 12.0 * p.nnz + 4.0 * (p.n + 1) + 16.0 * p.n * p.k
    ach = by / (kern["spmm_csr"] * 1e-3) / 1e9
    return {"kernel": "spmm_csr", "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "per_launch_alg": f"A + X + W = {by:.4g} bytes", "peak_source": src}


def cpu_baseline(name, budget_s=25.0, one_core=True):
    """The oracle as it stands, on the host cores, on a bounded sample of the workload: the config
    itself at FULL size (A built on the GPU by synth, copied to the host), timed per oracle sweep with
    a wall clock, median over as many sweeps as fit the budget (at least one; cfg3 ~3.4 s per sweep
    on 16 cores, cfg5 ~34 s).  one_core: also cfg1 / cfg2 with a single OpenMP thread."""
    import oracle
    import synth
    import torch
    p = synth.make_config(name, device="cuda" if name == "cfg3" and torch.cuda.is_available() else "cpu")
    if p.kind == "dense":
        op = oracle.Operator(A=p.A.cpu().numpy())
    else:
        op = oracle.Operator(row_ptr=p.row_ptr.cpu().numpy(), col_idx=p.col_idx.cpu().numpy(),
                             val=p.val.cpu().numpy())
    X = p.X0.cpu().numpy()
    del p
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        r = oracle.sweep(op, X)
        times.append(time.perf_counter() - t0)
        X = r.X
        if time.perf_counter() - t_start > budget_s or len(times) >= 20:
            break
    sec = statistics.median(times)
    out = {"value": 1.0 / sec, "unit": "sweeps/s", "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"{name} at full size from X0, {len(times)} consecutive oracle sweeps (median), "
                     f"{budget_s:.0f}s budget", "oracle_s_per_sweep": sec, "sample_sweeps": len(times),
           "affinity_cores": len(os.sched_getaffinity(0)), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}
    if one_core:
        code = ("import time,statistics,sys,oracle,synth;r={}\n"
                "for c in ('cfg1','cfg2'):\n"
                " p=synth.make_config(c);op=oracle.Operator(A=p.A.numpy());X=p.X0.numpy();ts=[]\n"
                " for _ in range(5 if c=='cfg2' else 50):\n"
                "  t=time.perf_counter();X=oracle.sweep(op,X).X;ts.append(time.perf_counter()-t)\n"
                " r[c]=1.0/statistics.median(ts)\n"
                "print(r, oracle.num_threads())")
        try:
            env = dict(os.environ, OMP_NUM_THREADS="1", PYTHONPATH=ROOT)
            o = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True, text=True,
                               timeout=120).stdout.strip().rsplit(" ", 1)
            import ast
            out["one_core_sweeps_s"] = ast.literal_eval(o[0])
            out["one_core_threads"] = int(o[1])
        except Exception as e:
            out["one_core_sweeps_s"] = {"error": repr(e)}
    return out


def run_reference(args, world, rank):
    """--impl reference: the oracle (plain CPU FP64 program) timed as it stands."""
    if rank != 0:
        return
    cb = cpu_baseline(args.config, budget_s=max(5.0, 150.0 / max(args.steps + args.warmup, 1)), one_core=False)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "sweeps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config}, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip per_config and cpu_baseline")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    hbm, hbm_src, fp64 = peaks()
    # Multi-GPU: A and X^ row-partitioned over the N ranks (NCCL over NVLink, DESIGN.md
    # "Multi-GPU"); one step = one sweep of the whole problem, so value = 1 / max-over-ranks time
    # (strong scaling).
    p = make_problem(args.config, f"cuda:{local}")
    with Clocks(local) as clk:
        ms, kern, R, X, st, s, ms_prof = time_ours(p, args.steps, args.warmup, world, local, rank=rank)
    ms_max = max_over_ranks(ms, world)
    value = 1000.0 / ms_max
    f, b = alg_counts(p)
    line = {"metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "n": p.n, "k": p.k, "kind": p.kind,
                       "nnz": p.nnz, "parallelism": f"rows{world}" if world > 1 else "single",
                       "l2": "inputs larger than L2 (A = %.2f GB)" % (p.nnz * 8 / 1e9) if p.kind == "dense"
                       else "A + X^ + W larger than L2"},
            "clocks": clk.summary(),
            "sweep": {"tflops_alg": f / (ms_max * 1e-3) / 1e12, "gbs_alg": b / (ms_max * 1e-3) / 1e9,
                      "frac_of_sweep_roofline": max(f / (fp64 * 1e12), b / (hbm * 1e9)) / (ms_max * 1e-3),
                      "F_alg": f, "B_alg": b, "status": s, "rel_resid": st.rel_resid, "corr_norm": st.corr_norm},
            "timing": "value: CUDA-graph replay of the sweep (collectives included at N > 1)" +
                      ", no instrumentation; kernels_ms: separate pass, direct launches with per-kernel CUDA events "
                      "(ms_per_step_instrumented)",
            "ms_per_step_instrumented": ms_prof,
            "kernels_ms": kern,
            "roofline": roofline_for(p, kern, ms_prof or ms_max, fp64, hbm, n_loc=partition(p.n, world, rank)[1] - partition(p.n, world, rank)[0]),
            "gpu_launches": R.kernels_per_sweep() * args.steps}
    if p.kind == "csr" and world == 1:
        line["s1_roofline"] = s1_roofline(p, kern)
    if world == 1:
        mx = time_mixed(p, local, max(3, args.steps // 2))
        if mx:
            line["mixed_next2"] = mx
        em = time_emul(p, local, max(3, args.steps // 2))
        if em:
            line["emul_ozaki"] = em
        rr_ms, rr_s = time_rr(R, X)
        line["rayleigh_ritz"] = {"ms": rr_ms, "status": rr_s, "what": "refine_rayleigh_ritz (NEXT-1, Sec. 3.4): "
                                 "S1 + pass B (D = 0) + k x k Cholesky/Jacobi + pass C + normalise"}
    # e2e through the host-buffer C ABI call
    e2e_s, h2d, d2h = time_e2e(R, p, max(3, args.steps // 2), 1, world, rank)
    e2e_s = max_over_ranks(e2e_s, world)
    line["e2e"] = {"value": 1.0 / e2e_s, "unit": "sweeps/s", "h2d_bytes_per_step": h2d * world,
                   "d2h_bytes_per_step": d2h * world}
    del R, X
    if not args.no_extra and world == 1:
        per = {}
        for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
            if name == args.config:
                per[name] = {"sweeps_s": value / world, "roofline": line["roofline"],
                             "frac_of_sweep_roofline": line["sweep"]["frac_of_sweep_roofline"]}
                continue
            q = make_problem(name, f"cuda:{local}")
            qms, qk, QR, QX, qst, qs, qprof = time_ours(q, 5 if q.n > 10000 else 20, 3, 1, local)
            qf, qb = alg_counts(q)
            qrr, _ = time_rr(QR, QX)
            per[name] = {"sweeps_s": 1000.0 / qms, "ms_per_sweep": qms, "ms_per_sweep_instrumented": qprof,
                         "rayleigh_ritz_ms": qrr,
                         "kernels_ms": qk, "roofline": roofline_for(q, qk, qprof or qms, fp64, hbm),
                         "s1_roofline": s1_roofline(q, qk),
                         "frac_of_sweep_roofline": max(qf / (fp64 * 1e12), qb / (hbm * 1e9)) / (qms * 1e-3)}
            del QR, QX
            torch.cuda.empty_cache()
            mx = time_mixed(q, local)
            if mx:
                per[name]["mixed_next2"] = mx
            em = time_emul(q, local)
            if em:
                per[name]["emul_ozaki"] = em
            del q
            torch.cuda.empty_cache()
        line["per_config"] = per
    if rank == 0 and world == 1 and not args.no_extra and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config)
        except Exception as e:  # never fail the bench on the baseline leg
            line["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
