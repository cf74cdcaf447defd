"""Per-launch sequence (library launch timing) of one TFT and one ITFT:
python tools/launch_seq.py C5 [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N, L, z, n, _ = bench.CONFIGS[cfg]
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
view = cf.DeviceView(dev)
for rep in range(reps):
    for name, fn in (("TFT", lambda: cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), view)),
                     ("ITFT", lambda: cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), view))):
        cf.launch_timing_read()
        cf.set_launch_timing(True)
        fn()
        cf.set_launch_timing(False)
        recs = cf.launch_timing_read()
        if rep == reps - 1:
            tot = sum(r[2] for r in recs)
            print(f"{cfg} {name}: {len(recs)} launches, {tot:.3f} ms")
            for k, b, ms in recs:
                print(f"  {k:28s} {ms:8.3f} ms  {b / 1e9:7.3f} GB alg  {b / max(ms, 1e-9) / 1e6:8.1f} GB/s")
