"""Opcode histogram of an ncu source page (sass) per work unit.
usage: python tools/sass_ops.py sass.csv UNITS"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ci = hdr.index("Instructions Executed")
si = hdr.index("Source")
units = float(sys.argv[2])
c = collections.Counter()
tot = 0
for r in data:
    s = r[si].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    n = int(r[ci] or 0)
    tot += n
    c[op] += n
print("per unit total", tot / units)
for op, n in c.most_common(45):
    print(f"{op:28s} {n / units:8.1f}  {n / tot * 100:5.2f}%")
