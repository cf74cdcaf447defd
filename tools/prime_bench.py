"""The reference's own ring (Goldilocks) on the GPU vs the unmodified reference
on one host core: TFT + ITFT at L = 2^22, z = n = 3 000 000 (seeded)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402
import pyoracle as po  # noqa: E402

P, m = cf.GOLDILOCKS, 32
L, z = 1 << 22, 3_000_000
rng = np.random.default_rng(1)
a = np.zeros((L, 1), dtype=np.uint64)
a[:z, 0] = rng.integers(0, P, size=z, dtype=np.uint64)
byts = (bench.tft_bytes(64, L, z, z) + bench.itft_bytes(64, L, z, z, 0))  # B = 8 bytes per coefficient
ctx = cf.PrimeRingCtx()
dev = torch.from_numpy(a.view(np.int64)).cuda()
view = cf.DeviceView(dev)
for _ in range(2):
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), view)
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), view)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), view)
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), view)
e1.record()
torch.cuda.synchronize()
gms = e0.elapsed_time(e1) / reps
print(f"GPU  TFT+ITFT L=2^22 z=n=3e6: {gms:.3f} ms  {byts / gms / 1e6:.1f} GB/s (algorithmic, B = 8)")
if po.ref_available():
    buf = np.ascontiguousarray(a.copy())
    ptr = buf.ctypes.data_as(po.U64P)
    c = C.c_uint64(0)
    t = time.perf_counter()
    po.ref().ref_tft(P, m, L, 0, z, z, ptr, L, 0, 1, 0, C.byref(c))
    po.ref().ref_itft(P, m, L, 0, z, z, 0, ptr, L, 0, 1, 0, C.byref(c))
    cms = (time.perf_counter() - t) * 1e3
    print(f"reference cf_tft+cf_itft (1 core): {cms:.1f} ms  {byts / cms / 1e6:.3f} GB/s  -> GPU {cms / gms:.0f}x")
