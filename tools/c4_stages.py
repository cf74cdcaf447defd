"""C4 pipeline stage times (CUDA events, warmed clocks): where poly_mul's time goes."""
import sys

import numpy as np
import torch

sys.path[:0] = [".", "oracle", "tests"]
import pyoracle as po  # noqa: E402
from helpers import to_dev  # noqa: E402

import paper_0810_3203_b200 as cf  # noqa: E402
from paper_0810_3203_b200 import polymul as pm  # noqa: E402

rng = np.random.default_rng(po.mix_seed(42, 4))
x = rng.integers(0, 1 << 64, size=(60000, 16), dtype=np.uint64, endpoint=False)
x[:, -1] &= np.uint64((1 << 40) - 1)
F = to_dev(x)
G = to_dev(x[::-1].copy())
for _ in range(3):
    pm.ss_mul(F, G, 1000)
torch.cuda.synchronize()
ctx = pm._fermat_ring(65536)  # the pipeline's cached context (plans warm)
W = ctx.element_words
zf = zg = 60000
n = zf + zg - 1
L = 1 << 17
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    ev[0].record()
    g = torch.zeros((L, W), dtype=torch.int64, device="cuda")
    h = torch.zeros((L, W), dtype=torch.int64, device="cuda")
    g[:zf, :16] = F
    h[:zg, :16] = G
    ev[1].record()
    cf.cf_tft(ctx, cf.TransformParams(L, 0, zf, n), cf.DeviceView(g))
    ev[2].record()
    cf.cf_tft(ctx, cf.TransformParams(L, 0, zg, n), cf.DeviceView(h))
    ev[3].record()
    pm.pointwise(ctx, g, h, n)
    ev[4].record()
    cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), cf.DeviceView(g))
    ev[5].record()
    cf.scale(ctx, cf.DeviceView(g), n, ctx.root_order() - 17)
    ev[6].record()
torch.cuda.synchronize()
names = ["setup", "tft g", "tft h", "pointwise", "itft", "scale"]
for i, nm in enumerate(names):
    print(f"{nm:10s} {ev[i].elapsed_time(ev[i + 1]):8.3f} ms")
print(f"total      {ev[0].elapsed_time(ev[6]):8.3f} ms")
