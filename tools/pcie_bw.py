"""Pinned host <-> HBM copy bandwidth on this box: H2D, D2H, both at once."""
import time

import torch

n = 3_280_000_000 // 8
h_in = torch.empty(n, dtype=torch.int64).pin_memory()
h_out = torch.empty(n, dtype=torch.int64).pin_memory()
d0 = torch.empty(n, dtype=torch.int64, device="cuda")
d1 = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d0.copy_(h_in, non_blocking=True)
    torch.cuda.synchronize()
    a = time.perf_counter() - t
    t = time.perf_counter()
    h_out.copy_(d1, non_blocking=True)
    torch.cuda.synchronize()
    b = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1):
        d0.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d1, non_blocking=True)
    torch.cuda.synchronize()
    c = time.perf_counter() - t
    gb = n * 8 / 1e9
    print(f"H2D {gb / a:6.1f} GB/s  D2H {gb / b:6.1f} GB/s  both {gb / c:6.1f} GB/s each")
