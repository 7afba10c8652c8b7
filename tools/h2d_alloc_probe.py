"""Split the cost of DenseTensor.to_device for a large pinned tensor: device allocation vs the copy."""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 68.7
n = int(gb * 1e9 / 8)
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
host.fill_(1.0)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: alloc {1e3 * (t1 - t0):7.1f} ms  copy {1e3 * (t2 - t1):7.1f} ms ({8 * n / (t2 - t1) / 1e9:.1f} GB/s)",
          flush=True)
    del dev
    torch.cuda.empty_cache()
t0 = time.perf_counter()
d2 = host.to("cuda")
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f".to(cuda) {1e3 * (t1 - t0):7.1f} ms ({8 * n / (t1 - t0) / 1e9:.1f} GB/s)")
