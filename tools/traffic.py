"""profiles/traffic.json from an ncu launch list of one TFT + one ITFT of a
config (the `--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` pass): per kernel name, the DRAM bytes per launch;
the whole step's DRAM bytes; and the sha256 of the library's sources, so that
bench.py reports the figures only for a build of the same sources.

usage: python tools/traffic.py CONFIG launches.csv [more.csv ...]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0810_3203_b200._build import source_sha256  # noqa: E402


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rows[1:]:
        name = r[ik].split("(")[0].split("<")[0].replace("void ", "").strip()
        d.setdefault((path, int(r[ii]), name), {})[r[im]] = float(r[iv].replace(",", ""))
    return d


def main():
    cfg, paths = sys.argv[1], sys.argv[2:]
    per, step, step_ms = {}, 0.0, 0.0
    for path in paths:
        for (_, _, name), v in sorted(launches(path).items()):
            b = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
            k = per.setdefault(name, {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
            k["launches"] += 1
            k["dram_bytes"] += b
            k["ms"] += v.get("gpu__time_duration.sum", 0) / 1e6
            step += b
            step_ms += v.get("gpu__time_duration.sum", 0) / 1e6
    for k in per.values():
        k["dram_bytes_per_launch"] = k["dram_bytes"] / k["launches"]
        k["share_of_step"] = k["ms"] / step_ms if step_ms else None
    out_path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        allc = json.load(open(out_path))
    except Exception:
        allc = {}
    allc = {k: v for k, v in allc.items() if isinstance(v, dict)}
    allc[cfg] = {"source_sha256": source_sha256(),
                 "step_dram_bytes": step, "step_ms_serialised": step_ms, "per_kernel": per,
                 "source": [os.path.relpath(p, ROOT) for p in paths],
                 "note": "ncu --clock-control none, one TFT + one ITFT: per-launch times are cold-cache and "
                         "serialised; bench.py uses the byte counts, its own CUDA events give the times"}
    json.dump(allc, open(out_path, "w"), indent=1)
    print(json.dumps(allc[cfg], indent=1))


if __name__ == "__main__":
    main()
