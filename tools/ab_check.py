"""Digest of GPU results on fixed seeded inputs (for A/B of experiment
builds): python tools/ab_check.py -> one line of sha1 prefixes."""
import hashlib
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0810_3203_b200 as cf  # noqa: E402

out = []
for (N, L, z, n, s) in ((131072, 1 << 18, 200000, 200000, 0), (131072, 1 << 18, 150001, 190000, 3),
                        (32768, 1 << 16, 65535, 65535, 0), (32768, 1 << 16, 40000, 50001, 5),
                        (8192, 4096, 3000, 3000, 0)):
    ctx = cf.FermatRingCtx(N)
    W = ctx.element_words
    g = torch.Generator(device="cuda").manual_seed(1234)
    dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
    dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda", generator=g)
    view = cf.DeviceView(dev)
    cf.cf_tft(ctx, cf.TransformParams(L, s, z, n), view)
    torch.cuda.synchronize()
    h1 = hashlib.sha1(dev[:n].cpu().numpy().tobytes()).hexdigest()[:10]
    dev[n:] = 0
    cf.cf_itft(ctx, cf.TransformParams(L, s, n, n, 0), view)
    torch.cuda.synchronize()
    h2 = hashlib.sha1(dev[:n].cpu().numpy().tobytes()).hexdigest()[:10]
    out.append(f"{h1}/{h2}")
print("digest", " ".join(out))
