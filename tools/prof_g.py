"""Runs ONE G-shape transform (Goldilocks, L = 2^22, z = n = 3e6) for ncu:
python tools/prof_g.py [tft|itft]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0810_3203_b200 as cf  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "tft"
L, z = 1 << 22, 3_000_000
rng = np.random.default_rng(1)
a = np.zeros((L, 1), dtype=np.uint64)
a[:z, 0] = rng.integers(0, cf.GOLDILOCKS, size=z, dtype=np.uint64)
ctx = cf.PrimeRingCtx()
dev = torch.from_numpy(a.view(np.int64)).cuda()
view = cf.DeviceView(dev)
if which == "tft":
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), view)
else:
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), view)
torch.cuda.synchronize()
print("done", which)
