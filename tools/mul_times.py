"""Times the BASELINE multiplication pipelines on the GPU (device-resident
inputs; CUDA events): C3 Nussbaumer negacyclic product, C4 SS Z[x] product."""
import sys

import numpy as np
import torch

sys.path[:0] = [".", "oracle", "tests"]
import pyoracle as po  # noqa: E402
from helpers import random_modulus, to_dev  # noqa: E402

from paper_0810_3203_b200 import polymul as pm  # noqa: E402


def timed(fn, reps=5, warm=5):
    for _ in range(warm):  # clocks ramp from idle: warm up before timing
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


K = s = 1024
m = random_modulus(po.mix_seed(42, 3))
rng = np.random.default_rng(po.mix_seed(42, 3))
f = to_dev(rng.integers(0, m, size=(K * s, 1), dtype=np.uint64)).view(-1)
g = to_dev(rng.integers(0, m, size=(K * s, 1), dtype=np.uint64)).view(-1)
print(f"C3 Nussbaumer negacyclic product, 2^20 terms mod 62-bit m: {timed(lambda: pm.nussbaumer_negacyclic_mul(f, g, m, K, s)):.2f} ms")
rng = np.random.default_rng(po.mix_seed(42, 4))


def limbs(count, bits):
    x = rng.integers(0, 1 << 64, size=(count, (bits + 63) // 64), dtype=np.uint64, endpoint=False)
    x[:, -1] &= np.uint64((1 << (bits % 64)) - 1)
    return x


F, G = to_dev(limbs(60000, 1000)), to_dev(limbs(60000, 1000))
print(f"C4 SS Z[x] product, 60000 x 1000-bit terms: {timed(lambda: pm.ss_mul(F, G, 1000)):.2f} ms")
