"""Pinned host<->device copy bandwidth on this box (context for e2e numbers)."""
import torch

for mb in (1, 16, 134):
    n = mb * (1 << 20) // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    h2d = 10 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    d2h = 10 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
    print(f"{mb:4d} MB: H2D {h2d:6.1f} GB/s  D2H {d2h:6.1f} GB/s")
