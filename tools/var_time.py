"""Per-call TFT / ITFT times over many repetitions (variance check)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
N, L, z, n, _ = bench.CONFIGS[cfg]
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
v = cf.DeviceView(dev)
tt, ti = [], []
for k in range(reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), v)
    e[1].record()
    cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), v)
    e[2].record()
    torch.cuda.synchronize()
    tt.append(e[0].elapsed_time(e[1]))
    ti.append(e[1].elapsed_time(e[2]))
print(cfg, "tft", " ".join("%.1f" % x for x in tt))
print(cfg, "itft", " ".join("%.1f" % x for x in ti))
