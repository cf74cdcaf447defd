"""One TFT (or ITFT) of an arbitrary Fermat shape, repeated (for ncu / timing):
python tools/prof_shape.py N L z n [tft|itft] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_0810_3203_b200 as cf  # noqa: E402

N, L, z, n = (int(x) for x in sys.argv[1:5])
which = sys.argv[5] if len(sys.argv) > 5 else "tft"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 1
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
view = cf.DeviceView(dev)
p = cf.TransformParams(L, 0, z, n) if which == "tft" else cf.TransformParams(L, 0, n, n, 0)
f = cf.cf_tft if which == "tft" else cf.cf_itft
for _ in range(2):
    f(ctx, p, view)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    f(ctx, p, view)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"N={N} L={L} z={z} n={n} {which}: {ms:.3f} ms, {ctx.element_bytes * L / 1e6:.1f} MB buffer")
