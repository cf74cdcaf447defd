"""Bucket a sass_lines_inner.py listing by enclosing function of wave_tma.cuh.
usage: python tools/sass_funcs.py lines.txt ITEMS"""
import collections
import re
import sys

src = open('paper_0810_3203_b200/csrc/wave_tma.cuh').read().split('\n')
bounds = [(i, l[:70]) for i, l in enumerate(src, 1) if re.match(r'^(__device__|__global__|template|struct)', l)]


def fn(ln):
    best = '?'
    for i, l in bounds:
        if i <= ln:
            best = l
    return best


items = float(sys.argv[2])
b = collections.Counter()
for l in open(sys.argv[1]).read().split('\n')[1:]:
    m = re.match(r'(\S+):(\d+)\s+([\d.]+)M', l)
    if not m:
        continue
    f, ln, n = m.group(1), int(m.group(2)), float(m.group(3))
    b[f if f != 'wave_tma.cuh' else fn(ln)] += n
for k, v in b.most_common(25):
    print(f"{v:8.1f}M {v * 1e6 / items:7.0f}/item  {k}")
