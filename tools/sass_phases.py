"""Attribute ncu per-instruction counts/stalls to kernel source lines, using the
outermost inlining site (nvdisasm -gi), and bucket them by phase ranges.

usage: python tools/sass_phases.py ncu_sass.csv nvdisasm_gi.sass symbol [start:end:name ...]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ci = hdr.index("Instructions Executed")
wi = hdr.index("Warp Stall Sampling (All Samples)")
sym = sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    s, e, n = a.split(":")
    ranges.append((int(s), int(e), n))
lines = open(sys.argv[2]).read().split("\n")
start = [k for k, l in enumerate(lines) if l.startswith(".text." + sym + ":")][0]
cur = None
mapping = []
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    if "//## File" in l:
        nums = re.findall(r'line (\d+)', l)
        cur = int(nums[-1]) if nums else None
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        mapping.append(cur)
assert len(mapping) == len(data), (len(mapping), len(data))
agg, st = collections.Counter(), collections.Counter()
for r, ln in zip(data, mapping):
    name = "other"
    for s, e, n in ranges:
        if ln is not None and s <= ln <= e:
            name = n
    agg[name] += float(r[ci] or 0)
    st[name] += float(r[wi] or 0)
T, S = sum(agg.values()), sum(st.values())
for n in sorted(agg, key=lambda k: -agg[k]):
    print(f"{n:12s} {agg[n]:14.0f} inst {100 * agg[n] / T:6.2f}%   stall {100 * st[n] / S:6.2f}%")
