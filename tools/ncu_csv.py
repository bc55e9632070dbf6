"""Compact view of an `ncu --metrics ... --csv` log: one line per kernel launch (first of repeats)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
d = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        key = (x["Kernel Name"].split("(")[0][:48], x["Grid Size"])
        if key in d and x["ID"] != d[key]["id"]:
            continue
        e = d.setdefault(key, {"id": x["ID"]})
        try:
            e[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
        except ValueError:
            pass
short = {"gpu__time_duration.sum": ("t_us", 1e-3), "dram__bytes_read.sum": ("dramR_GB", 1e-9),
         "dram__bytes_write.sum": ("dramW_GB", 1e-9), "lts__t_bytes.sum": ("lts_GB", 1e-9)}
for k, v in d.items():
    parts = []
    for m, val in v.items():
        if m == "id":
            continue
        name, sc = short.get(m, (m.split("__")[1][:22] if "__" in m else m, 1.0))
        parts.append(f"{name}={val * sc:.3g}")
    print(f"{k[0]:48s} {k[1]:12s} " + " ".join(parts))
