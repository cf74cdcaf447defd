import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_0810_3203_b200 as cf
import bench
N, L, z, n, _ = bench.CONFIGS['C1']
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
a = np.zeros((L, W), dtype=np.uint64)
rng = np.random.default_rng(1)
a[:z, :N//64] = rng.integers(0, 1<<63, size=(z, N//64), dtype=np.uint64)
dev = torch.from_numpy(a.view(np.int64)).cuda()
view = cf.DeviceView(dev)
def rt():
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), view)
    cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), view)
for _ in range(5): rt()
torch.cuda.synchronize()
for which in ('tft','itft','rt'):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        if which == 'tft': cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), view)
        elif which == 'itft': cf.cf_itft(ctx, cf.TransformParams(L, 0, n, n, 0), view)
        else: rt()
    e1.record(); torch.cuda.synchronize()
    print(which, round(e0.elapsed_time(e1) / 50 * 1000, 1), 'us')
