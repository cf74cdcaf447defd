"""Per-source-line (innermost inlined location) warp-instruction counts of
one kernel from an ncu SASS source page and an nvdisasm -gi listing.
usage: python tools/sass_lines_inner.py sass.csv disasm.txt SYMBOL [N]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ci = hdr.index("Instructions Executed")
si = hdr.index("Source")
lines = open(sys.argv[2]).read().split("\n")
sym = sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 60
start = [k for k, l in enumerate(lines) if l.startswith(".text." + sym + ":")][0]
cur, fresh, mapping = None, True, []
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    if "//## File" in l:
        fm = re.search(r'File "([^"]+)", line (\d+)', l)
        if fm and fresh:
            cur = f"{fm.group(1).split('/')[-1]}:{fm.group(2)}"
            fresh = False
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        mapping.append(cur)
        fresh = True
c, ops = collections.Counter(), collections.defaultdict(collections.Counter)
tot = 0
for r, src in zip(data, mapping):
    n = int(r[ci] or 0)
    s = r[si].strip().split()
    op = (s[1] if s and s[0].startswith("@") else (s[0] if s else "?")).split(".")[0]
    c[src] += n
    ops[src][op] += n
    tot += n
print(f"total {tot / 1e6:.1f}M warp instructions")
for s, n in c.most_common(top):
    mix = " ".join(f"{o}:{100 * k / max(n, 1):.0f}" for o, k in ops[s].most_common(4))
    print(f"{str(s):28s} {n / 1e6:8.1f}M {100 * n / tot:5.1f}%  {mix}")
