"""Micro-benchmark: device copy bandwidth vs working-set size (L2 vs HBM)."""
import torch

torch.cuda.set_device(0)
for mb in (8, 16, 32, 48, 64, 96, 128, 512, 2048):
    n = mb * (1 << 20) // 2
    a = torch.empty(n, dtype=torch.int16, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = max(5, int(4096 / mb))
    e0.record()
    for _ in range(it):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / it / 1e3
    print(f"copy {mb:5d} MiB (x2 = r+w): {2 * mb * (1 << 20) / t / 1e9:8.0f} GB/s")
