"""Runs ONE transform of a BASELINE config (for ncu): python tools/prof_one.py C5 [tft|itft]."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
which = sys.argv[2] if len(sys.argv) > 2 else "tft"
N, L, z, n, _ = bench.CONFIGS[cfg]
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
view = cf.DeviceView(dev)
if which == "tft":
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), view)
else:
    cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), view)
torch.cuda.synchronize()
print("done", cfg, which)
