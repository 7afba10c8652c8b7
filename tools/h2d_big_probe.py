"""H2D strategies for a large pinned host tensor: one copy vs chunks round-robin over streams."""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 68.7
n = int(gb * 1e9 / 8)
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
host.fill_(1.0)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def run(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{label:34s} {dt * 1e3:8.1f} ms  {8 * n / dt / 1e9:6.1f} GB/s", flush=True)


run("single copy_", lambda: dev.copy_(host, non_blocking=True))
for ns in (2, 4, 8):
    for chunk_mb in (256, 1024):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        chunk = chunk_mb * (1 << 20) // 8

        def f():
            for i, st in enumerate(range(0, n, chunk)):
                s = streams[i % ns]
                with torch.cuda.stream(s):
                    dev[st:st + chunk].copy_(host[st:st + chunk], non_blocking=True)
        run(f"{ns} streams x {chunk_mb} MiB chunks", f)
