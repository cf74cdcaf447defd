"""G shape (Goldilocks, L = 2^22, z = n = 3e6): TFT / ITFT device time per
leaf limit, and the library's per-launch timing of the default plan."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0810_3203_b200 as cf  # noqa: E402

P = cf.GOLDILOCKS
L, z = 1 << 22, 3_000_000
rng = np.random.default_rng(1)
a = np.zeros((L, 1), dtype=np.uint64)
a[:z, 0] = rng.integers(0, P, size=z, dtype=np.uint64)
ctx = cf.PrimeRingCtx()
dev = torch.from_numpy(a.view(np.int64)).cuda()
view = cf.DeviceView(dev)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tft = lambda: cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), view)  # noqa: E731
itft = lambda: cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), view)  # noqa: E731
for lim in [int(x) for x in sys.argv[1:]] or [0, 4, 5, 6, 7, 8, 9, 10]:
    got = ctx.set_leaf_limit(lim)
    print(f"leaf_limit {lim} (max ell {got}): TFT {timeit(tft):.3f} ms  ITFT {timeit(itft):.3f} ms", flush=True)
ctx.set_leaf_limit(0)
cf.set_launch_timing(True)
tft()
itft()
torch.cuda.synchronize()
for r in cf.launch_timing_read():
    print(r)
cf.set_launch_timing(False)
