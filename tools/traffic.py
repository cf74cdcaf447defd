"""Per-launch DRAM traffic and time from an ncu --csv metrics log:
python tools/traffic.py gpurun_out/x.csv"""
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rows[1:]:
        d.setdefault((int(r[ii]), r[ik][:28]), {})[r[im]] = float(r[iv].replace(",", ""))
    tb = tt = 0.0
    for k, v in sorted(d.items()):
        rd, wr = v.get("dram__bytes_read.sum", 0) / 1e9, v.get("dram__bytes_write.sum", 0) / 1e9
        t = v.get("gpu__time_duration.sum", 0) / 1e6
        tb += rd + wr
        tt += t
        print(f"{k[0]:3d} {k[1]:28s} rd {rd:6.2f} wr {wr:6.2f} GB  {t:7.3f} ms  {(rd + wr) / t if t else 0:6.2f} TB/s")
    print(f"{path}: {tb:.2f} GB in {tt:.3f} ms")
