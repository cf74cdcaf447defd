"""One C4 Schoenhage-Strassen product after warm-up (for ncu launch lists)."""
import sys

import numpy as np
import torch

sys.path[:0] = [".", "oracle", "tests"]
import pyoracle as po  # noqa: E402
from helpers import to_dev  # noqa: E402

from paper_0810_3203_b200 import polymul as pm  # noqa: E402

rng = np.random.default_rng(po.mix_seed(42, 4))


def limbs(count, bits):
    x = rng.integers(0, 1 << 64, size=(count, (bits + 63) // 64), dtype=np.uint64, endpoint=False)
    x[:, -1] &= np.uint64((1 << (bits % 64)) - 1)
    return to_dev(x)


F, G = limbs(60000, 1000), limbs(60000, 1000)
for _ in range(3):
    pm.ss_mul(F, G, 1000)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pm.ss_mul(F, G, 1000)
e1.record()
torch.cuda.synchronize()
print("C4 ms", e0.elapsed_time(e1))
