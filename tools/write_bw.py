"""Measured HBM write-only and read-only bandwidth (torch fill / sum over 4 GiB), the
rooflines for the write-dominated tile pass and the read-dominated passes."""
import torch

n = 1 << 29  # 4 GiB of fp64
x = torch.empty(n, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (("write-only (fill_)", lambda: x.fill_(1.0), 8 * n),
                         ("read-only (sum)", lambda: x.sum(), 8 * n),
                         ("copy (read + write)", lambda: x[: n // 2].copy_(x[n // 2:]), 8 * n)):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {nbytes / best / 1e6:.0f} GB/s")
