"""Measure the FP64 roofline denominators on the GPU box (cuBLAS DGEMM via torch, plus
tools/fp64_peak DMMA/DFMA microbenchmarks run separately). Output: one JSON line."""
import json, os, time, subprocess, torch
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best
out = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
try:
    out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception:
    pass
d = "cuda"
for (m, n, k) in [(8192, 8192, 8192), (32768, 64, 32768), (4096, 16, 4096), (128, 128, 4096000 // 4)]:
    a = torch.randn(m, k, dtype=torch.float64, device=d)
    b = torch.randn(k, n, dtype=torch.float64, device=d)
    s = t(lambda: a @ b)
    out[f"dgemm_{m}x{n}x{k}_tflops"] = 2 * m * n * k / s / 1e12
    del a, b
x = torch.empty(2**30 // 8 * 4, dtype=torch.float64, device=d)
y = torch.empty_like(x)
s = t(lambda: y.copy_(x))
out["copy_gbs"] = 2 * x.numel() * 8 / s / 1e9
print(json.dumps(out))
