"""Pinned H2D bandwidth as a function of buffer size (one copy per size)."""
import time

import torch

for gb in (1, 4, 8, 16, 32, 48, 68):
    n = int(gb * (1 << 30) / 8)
    host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    host.fill_(1.0)
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(2):
        t0 = time.perf_counter()
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, 8 * n / (time.perf_counter() - t0) / 1e9)
    # the same bytes as 1 GiB pieces of the big buffer
    t0 = time.perf_counter()
    step = (1 << 30) // 8
    for s in range(0, n, step):
        dev[s:s + step].copy_(host[s:s + step], non_blocking=True)
    torch.cuda.synchronize()
    pieces = 8 * n / (time.perf_counter() - t0) / 1e9
    print(f"{gb:3d} GiB pinned: {best:6.1f} GB/s one copy, {pieces:6.1f} GB/s in 1 GiB pieces", flush=True)
    del host, dev
    torch.cuda.empty_cache()
