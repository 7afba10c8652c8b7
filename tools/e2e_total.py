"""Wall time of the end-to-end call nncp_sequential(DenseTensor(pinned host tensor)) at a BASELINE shape."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
R = int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
fs = truth_factors(dims, R, 1, "uniform")
xd = synthetic_block(dims, fs, 0.01, 1)
host = torch.empty(xd.numel(), dtype=torch.float64, pin_memory=True)
host.copy_(xd)
del xd
torch.cuda.empty_cache()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = P.nncp_sequential(P.DenseTensor(dims, host), P.RunConfig(rank=R, algorithm="hals", max_iters=steps, tol=0.0))
    torch.cuda.synchronize()
    print(f"e2e {steps} iterations: {1e3 * (time.perf_counter() - t0):8.1f} ms  eps {r.errors[-1]:.6e}", flush=True)
    del r
    torch.cuda.empty_cache()
