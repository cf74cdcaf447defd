import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "tests"]
import numpy as np, torch
import pyoracle as po
from helpers import to_dev, from_dev
import paper_0810_3203_b200 as cf
from paper_0810_3203_b200 import polymul as pm
from concurrent.futures import ThreadPoolExecutor

N, L, zf, zg = 4096, 8192, 3000, 2500
n = zf + zg - 1
ctx = cf.FermatRingCtx(N); ring = po.Ring.fermat(N)
W = ctx.element_words; lim = N // 64
rng = np.random.default_rng(11)
A = np.zeros((L, W), np.uint64); B = np.zeros((L, W), np.uint64)
A[:zf, :8] = rng.integers(0, 1 << 64, size=(zf, 8), dtype=np.uint64, endpoint=False)
B[:zg, :8] = rng.integers(0, 1 << 64, size=(zg, 8), dtype=np.uint64, endpoint=False)
dA, dB = to_dev(A), to_dev(B)
def cmp(tag, dev, ref, k):
    g = from_dev(dev)
    bad = [i for i in range(k) if not np.array_equal(g[i, :lim + 1], ref[i, :lim + 1])]
    print(tag, "bad", len(bad), bad[:8], flush=True)
cf.cf_tft(ctx, cf.TransformParams(L, 0, zf, n), cf.DeviceView(dA)); ring.tft(A, L, 0, zf, n, threads=8)
cmp("tftA", dA, A, n)
cf.cf_tft(ctx, cf.TransformParams(L, 0, zg, n), cf.DeviceView(dB)); ring.tft(B, L, 0, zg, n, threads=8)
cmp("tftB", dB, B, n)
dA, dB = to_dev(A), to_dev(B)  # continue from the oracle state
pm.pointwise(ctx, dA, dB, n); cf.canonicalize(ctx, dA, n)
with ThreadPoolExecutor(8) as ex:
    P = list(ex.map(lambda i: ring.mul(A[i, :lim + 1], B[i, :lim + 1]), range(n)))
for i in range(n): A[i, :lim + 1] = P[i]
cmp("pointwise", dA, A, n)
dA = to_dev(A)
cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), cf.DeviceView(dA)); ring.itft(A, L, 0, n, n, 0, threads=8)
cmp("itft", dA, A, n)
dA = to_dev(A)
cf.scale(ctx, cf.DeviceView(dA), n, 2 * N - 13)
for i in range(n): A[i, :lim + 1] = ring.twiddle(2 * N - 13, A[i, :lim + 1])
cmp("scale", dA, A, n)
