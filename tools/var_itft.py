"""ITFT-only repetitions (outlier hunt): python tools/var_itft.py C5 30"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
N, L, z, n, _ = bench.CONFIGS[cfg]
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
v = cf.DeviceView(dev)
ts = []
for k in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), v)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    print("itft %d %.1f ms" % (k, ts[-1]), file=sys.stderr, flush=True)
print(cfg, "itft", " ".join("%.1f" % x for x in ts))
