"""Steady-state TFT / ITFT times of one config under each engine mode.

usage: python tools/mode_time.py C5 [wide ...]   (wide: 0 radix-8 waves, 1 radix-64 CTA waves)
"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
modes = [int(x) for x in sys.argv[2:]] or [0, 1]
N, L, z, n, _ = bench.CONFIGS[cfg]
dev = None
for wide in modes:
    ctx = cf.FermatRingCtx(N)
    ctx.set_wide(wide)
    W = ctx.element_words
    if dev is None:
        dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
        dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
    v = cf.DeviceView(dev)
    best = None
    for k in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), v)
        e[1].record()
        cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), v)
        e[2].record()
        torch.cuda.synchronize()
        t = (e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]))
        if k >= 2 and (best is None or sum(t) < sum(best)):
            best = t
    gb = (bench.tft_bytes(N, L, z, n) + bench.itft_bytes(N, L, n, n, 0)) / 1e9
    print(f"{cfg} wide={wide} tft {best[0]:.3f} ms itft {best[1]:.3f} ms  {gb / (sum(best) / 1e3):.1f} GB/s", flush=True)
