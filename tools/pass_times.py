"""Times the top-level passes of a BASELINE transform separately (batched
sub-transforms through cftft_gpu_batch): python tools/pass_times.py C5"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_0810_3203_b200 as cf  # noqa: E402
from paper_0810_3203_b200.dist import Sub  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
N, L, z, n, _ = bench.CONFIGS[cfg]
ctx = cf.FermatRingCtx(N)
W = ctx.element_words
dev = torch.zeros((L, W), dtype=torch.int64, device="cuda")
dev[:z, : N // 64] = torch.randint(-(1 << 62), 1 << 62, (z, N // 64), device="cuda")
B = N // 8
for name, inv, subs in bench.bailey_phases(2 * N, L, z, n, 0, False) + bench.bailey_phases(2 * N, L, n, n, 0, True):
    items = [Sub(*t) for t in subs]
    byts = B * sum(t[2] + t[3] + t[4] for t in subs)
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cf.run_batch(ctx, inv, items, dev)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{cfg} {name:12s} subs {len(items):4d}  {ms:8.3f} ms  {byts / ms / 1e6:8.1f} GB/s (algorithmic)", flush=True)
