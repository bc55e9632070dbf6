"""Per-kernel summary of an ncu report: duration, DMMA utilisation, occupancy, stall breakdown,
and the SASS lines with the most stall samples.   python tools/ncu_stalls.py <rep> [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
h = raw[0]
for x in raw[2:]:
    d = dict(zip(h, x))
    print("==", d["Kernel Name"][:90])
    for k in ("gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum", "lts__t_bytes.sum",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"):
        if k in d:
            print(f"   {k} = {d[k]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v.replace('.', '', 1).isdigit()}
    tot = sum(st.values()) or 1
    print("   stalls:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(st.items(), key=lambda a: -a[1])[:9]))
src = list(csv.reader(run("--page", "source", "--csv", "--print-source", "sass").splitlines()))
idx = [j for j, x in enumerate(src) if x and x[0] == "Address"]
for n, i in enumerate(idx):
    hh = src[i]
    end = idx[n + 1] - 1 if n + 1 < len(idx) else len(src)
    rows = [dict(zip(hh, x)) for x in src[i + 1:end] if len(x) == len(hh)]

    def f(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    tot = sum(f(x["Warp Stall Sampling (All Samples)"]) for x in rows) or 1
    stalls = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
    print(f"-- kernel {n}: top SASS by stall samples")
    for x in sorted(rows, key=lambda x: -f(x["Warp Stall Sampling (All Samples)"]))[:top]:
        smp = f(x["Warp Stall Sampling (All Samples)"])
        st = sorted(((c[6:], f(x[c])) for c in stalls), key=lambda a: -a[1])[:2]
        print(f"   {x['Source'][:56]:56s} {smp / tot * 100:5.1f}%  exec={x['Instructions Executed']}  {st}")
