"""Summarise ncu outputs into small committed files under profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.json>
  python tools/ncu_summary.py report <prof.ncu-rep> <out.json> [name]
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0]
            v = float(d["Metric Value"].replace(",", ""))
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(
                d["Metric Unit"], 1.0)
            agg.setdefault(name, []).append(v * scale)
    skip = ("absrow_max_dense_kernel", "absrow_max_csr_kernel", "max_kernel", "col_range_kernel", "spmm_xoff_kernel")
    mine = ("gemm_ax", "w_finish", "kxk_", "passB", "passC", "norm_reduce", "normalize", "spmm_", "ag_local",
            "absrow_max", "max_kernel", "col_range")
    ours = {k: v for k, v in agg.items() if any(m in k.split("<")[0] for m in mine)}
    init = lambda k: any(x in k for x in skip)
    tot = sum(sum(v) / len(v) for k, v in ours.items() if not init(k))
    res = {"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised); "
                                  "per-kernel mean us per launch and share of the per-sweep kernel time",
           "kernels": {k: {"launches": len(v), "mean_us": sum(v) / len(v),
                           "share_of_sweep": (sum(v) / len(v)) / tot if not init(k) else None}
                       for k, v in ours.items()},
           "sweep_kernel_time_us": tot}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def report(path, out, name=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
            "sm__cycles_elapsed.avg.per_second"]
    res = {"source": path, "kernels": []}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        ent = {"kernel": d["Kernel Name"]}
        for k in keep:
            if k in d:
                ent[k] = f"{d[k]} {u[k]}".strip()
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
              if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k and v not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        ent["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        res["kernels"].append(ent)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        report(sys.argv[2], sys.argv[3])
