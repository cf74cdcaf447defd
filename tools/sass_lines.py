"""Attribute ncu per-instruction counts to source lines.

usage: python tools/sass_lines.py <ncu-sass.csv> <nvdisasm --print-line-info output> <kernel symbol>
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
lines = open(sys.argv[2]).read().split("\n")
start = None
for k, l in enumerate(lines):
    if l.startswith(".text." + sym + ":"):
        start = k
        break
cur = None
mapping = []  # source line per instruction
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    m = re.search(r'line (\d+)', l)
    if "//## File" in l:
        fm = re.search(r'File "([^"]+)", line (\d+)', l)
        if fm:
            cur = f"{fm.group(1).split('/')[-1]}:{fm.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        mapping.append(cur)
print("instructions: ncu", len(data), "disasm", len(mapping))
agg = collections.Counter()
st = collections.Counter()
for r, src in zip(data, mapping):
    agg[src] += float(r[ci] or 0)
    st[src] += float(r[wi] or 0)
tot = sum(agg.values())
tst = sum(st.values())
for src, v in agg.most_common(40):
    print(f"{src:40s} {100 * v / tot:6.2f}% inst {100 * st[src] / tst:6.2f}% stall")
