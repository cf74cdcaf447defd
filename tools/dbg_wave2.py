import os, sys
sys.path[:0] = [".", "oracle", "tests"]
import numpy as np
import pyoracle as po
from helpers import fermat_inputs, from_dev, to_dev
import paper_0810_3203_b200 as cf
N = 4096
ctx = cf.FermatRingCtx(N)
ring = po.Ring.fermat(N)
W = ctx.element_words; lim = N // 64; P = (1 << N) + 1
for (L, s, z, n, f) in [(16, 2273, 15, 4, 0), (16, 2272, 15, 4, 0), (16, 2304, 15, 4, 0)]:
    buf = fermat_inputs(N, L, z, W, 3)
    want = buf.copy(); ring.itft(want, L, s, z, n, f)
    dev = to_dev(buf); cf.cf_itft(ctx, cf.TransformParams(L, s, z, n, f), cf.DeviceView(dev)); got = from_dev(dev)
    for i in range(n + f):
        g = sum(int(got[i, k]) << (64 * k) for k in range(lim + 1)); w = sum(int(want[i, k]) << (64 * k) for k in range(lim + 1))
        d = (g - w) % P; dd = min(d, P - d)
        print(L, s, i, "ok" if d == 0 else f"diff bits {dd.bit_length()} tz {(dd & -dd).bit_length()-1} sign {'+' if d < P//2 else '-'} hex {hex(dd)[:24]}")
