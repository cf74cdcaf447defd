"""Attribute ncu per-instruction counts and stall samples to source lines
through the inline chains of `nvdisasm -gi` (outermost call site first).

  ncu -i X.ncu-rep --page source --csv > src.csv
  cuobjdump -xelf all libcftft_b200.so; nvdisasm -gi -c capi.sm_100a.cubin > gi.sass
  python tools/sass_attr.py src.csv gi.sass MANGLED_KERNEL_SYMBOL [DEPTH]

Prints, per chain prefix of DEPTH source lines: share of the instructions
executed, share of the stall samples, the top opcodes."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ci = hdr.index("Instructions Executed"); wi = hdr.index("Warp Stall Sampling (All Samples)")
si = hdr.index("Source")
sym = sys.argv[3]; depth = int(sys.argv[4]) if len(sys.argv) > 4 else 2
lines = open(sys.argv[2]).read().split("\n")
start = [k for k, l in enumerate(lines) if l.startswith(".text." + sym + ":")][0]
chain = []; mapping = []; fresh = True
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"): break
    if "//## File" in l:
        if fresh: chain = []; fresh = False
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        chain.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        mapping.append(tuple(chain)); fresh = True
assert len(mapping) == len(data), (len(mapping), len(data))
agg, st = collections.Counter(), collections.Counter()
ops = collections.defaultdict(collections.Counter)
for r, ch in zip(data, mapping):
    # chain: innermost first; dedupe "X inlined at Y" + "Y" pairs -> take lines outer->inner
    seq = []
    for f, ln in reversed(ch):
        if not seq or seq[-1] != (f, ln): seq.append((f, ln))
    key = tuple(f"{f.split('.')[0][-6:]}:{ln}" for f, ln in seq[:depth])
    n = float(r[ci] or 0)
    agg[key] += n; st[key] += float(r[wi] or 0)
    op = r[si].split()[0] if not r[si].startswith("@") else r[si].split()[1]
    ops[key][op.split(".")[0]] += n
T, S = sum(agg.values()), sum(st.values())
print("total inst", T, "samples", S)
for n in sorted(agg, key=lambda k: -agg[k]):
    if agg[n] / T < 0.004 and st[n] / S < 0.004: continue
    top = " ".join(f"{o}:{100*c/agg[n]:.0f}" for o, c in ops[n].most_common(5)) if agg[n] else ""
    print(f"{' > '.join(n):40s} {100 * agg[n] / T:6.2f}% inst  {100 * st[n] / S:6.2f}% stall   {top}")
