import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "tests"]
import numpy as np, torch
import pyoracle as po
from helpers import to_dev, from_dev
import paper_0810_3203_b200 as cf
from paper_0810_3203_b200 import polymul as pm

for N in [int(a) for a in sys.argv[1:]] or [2048, 4096, 8192, 16384]:
    ctx = cf.FermatRingCtx(N); ring = po.Ring.fermat(N)
    W = ctx.element_words; lim = N // 64
    rng = np.random.default_rng(N)
    cnt = 64
    a = np.zeros((cnt, W), np.uint64); b = np.zeros((cnt, W), np.uint64)
    a[:, :lim] = rng.integers(0, 1 << 64, size=(cnt, lim), dtype=np.uint64, endpoint=False)
    b[:, :lim] = rng.integers(0, 1 << 64, size=(cnt, lim), dtype=np.uint64, endpoint=False)
    a[1, :lim] = 0; a[1, :8] = rng.integers(0, 1 << 64, size=8, dtype=np.uint64, endpoint=False)
    b[1, :lim] = 0; b[1, :8] = rng.integers(0, 1 << 64, size=8, dtype=np.uint64, endpoint=False)
    da, db = to_dev(a), to_dev(b)
    pm.pointwise(ctx, da, db, cnt); cf.canonicalize(ctx, da, cnt)
    got = from_dev(da)
    bad = [i for i in range(cnt) if not np.array_equal(got[i, :lim + 1], ring.mul(a[i, :lim + 1], b[i, :lim + 1]))]
    print("pointwise N", N, "bad", bad[:10], len(bad))
    # pipeline stages for ss_mul-like shape
    L = 2048; zf = 1000
    A = np.zeros((L, W), np.uint64); A[:zf, :8] = rng.integers(0, 1 << 64, size=(zf, 8), dtype=np.uint64, endpoint=False)
    dA = to_dev(A); want = A.copy()
    cf.cf_tft(ctx, cf.TransformParams(L, 0, zf, 1999), cf.DeviceView(dA))
    ring.tft(want, L, 0, zf, 1999)
    g = from_dev(dA)
    print("tft bad rows", int(sum(not np.array_equal(g[i, :lim + 1], want[i, :lim + 1]) for i in range(1999))))
