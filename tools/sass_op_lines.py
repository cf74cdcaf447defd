"""Where one opcode's executions come from (by source line).
usage: python tools/sass_op_lines.py sass.csv disasm.txt SYMBOL OPCODE-PREFIX UNITS"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ci = hdr.index("Instructions Executed")
si = hdr.index("Source")
lines = open(sys.argv[2]).read().split("\n")
sym, want, units = sys.argv[3], sys.argv[4], float(sys.argv[5])
start = [k for k, l in enumerate(lines) if l.startswith(".text." + sym + ":")][0]
cur, mapping = None, []
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    if "//## File" in l:
        fm = re.search(r'File "([^"]+)", line (\d+)', l)
        if fm:
            cur = f"{fm.group(1).split('/')[-1]}:{fm.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        mapping.append(cur)
c = collections.Counter()
for r, src in zip(data, mapping):
    s = r[si].strip().split()
    if not s:
        continue
    op = s[1] if s[0].startswith("@") else s[0]
    if op.startswith(want):
        c[src] += int(r[ci] or 0)
for src, n in c.most_common(25):
    print(f"{str(src):36s} {n / units:8.1f}")
