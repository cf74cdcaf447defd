"""Per-launch summary of an ncu --csv metric list: python tools/launch_summary.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ix = {k: j for j, k in enumerate(h)}
k = collections.OrderedDict()
for r in rows[start + 1:]:
    key = (int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0][:34])
    v = r[ix["Metric Value"]].replace(",", "")
    k.setdefault(key, {})[r[ix["Metric Name"]]] = float(v) if v else 0.0
tot_t = 0
for (i, name), m in k.items():
    t = m.get("gpu__time_duration.sum", 0) / 1e6
    tot_t += t
    rd, wr = m.get("dram__bytes_read.sum", 0) / 1e9, m.get("dram__bytes_write.sum", 0) / 1e9
    inst = m.get("smsp__inst_executed.sum", 0) / 1e6
    lts = m.get("lts__t_bytes.sum", 0) / 1e9
    print(f"{i:3d} {name:34s} {t:7.3f} ms  dram r {rd:6.2f} w {wr:6.2f} GB ({(rd + wr) / max(t, 1e-9):5.2f} TB/s)"
          f"  L2 {lts:6.2f} GB  inst {inst:7.1f} M")
print(f"total {tot_t:.3f} ms")
