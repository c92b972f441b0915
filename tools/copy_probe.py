"""H2D copy time of a pinned 15 MB buffer: just written by the CPU vs not,
GPU idle vs busy (debug aid for the e2e topology copies)."""
import time
import numpy as np
import torch

n = 15 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
hn = h.numpy()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
big = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()


def timed(write, busy, gap_ms=0.0):
    torch.cuda.synchronize()
    if write:
        hn[:] = np.random.randint(0, 255, 1)[0]
    if gap_ms:
        time.sleep(gap_ms / 1e3)
    if busy:
        for _ in range(20):
            big.mul_(1.0000001)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for write in (False, True):
    for busy in (False, True):
        for gap in (0.0, 5.0):
            ts = [timed(write, busy, gap) for _ in range(8)][2:]
            print(f"written {write!s:5} gpu_busy {busy!s:5} gap {gap:3.0f} ms: "
                  f"{np.median(ts):.3f} ms  ({n / np.median(ts) / 1e6:.1f} GB/s)")

# concurrent with an atomic-heavy kernel on another stream (like k_raster_many)
idx = torch.randint(0, 1 << 24, (1 << 26,), device="cuda")
src = torch.randint(0, 1 << 20, (1 << 26,), device="cuda", dtype=torch.int32)
dst = torch.full((1 << 24,), 1 << 30, device="cuda", dtype=torch.int32)
k = torch.cuda.Stream()
for busy in (False, True):
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        if busy:
            with torch.cuda.stream(k):
                for _ in range(4):
                    dst.scatter_reduce_(0, idx, src, reduce="amin")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            d.copy_(h, non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"atomics on another stream {busy}: {np.median(ts[2:]):.3f} ms")
