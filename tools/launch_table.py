"""Per-launch table of an ncu --csv log (duration, DRAM bytes, GB/s): python tools/launch_table.py log.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
per = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "")[:26], d.get("Grid Size", ""))
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9}.get(u, 1)
    per.setdefault(k, {})[d["Metric Name"]] = v * scale
tt = tb = 0
for (i, name, grid), m in per.items():
    t = m.get("gpu__time_duration.sum", 0)
    b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tt += t
    tb += b
    print(f"{i:>4} {name:26s} {grid:>14s} {t * 1e3:8.3f} ms {b / 1e9:7.2f} GB {b / max(t, 1e-12) / 1e9:7.0f} GB/s")
print(f"total {tt * 1e3:.3f} ms, {tb / 1e9:.2f} GB, {tb / max(tt, 1e-12) / 1e9:.0f} GB/s")
