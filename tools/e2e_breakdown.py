"""Phase timing of the end-to-end call nncp_sequential(DenseTensor(pinned host tensor)) at a BASELINE config."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import driver as D  # noqa: E402
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
torch.cuda.synchronize()


def mark(label, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"{label:28s} {1e3 * (t - t0):9.1f} ms", flush=True)
    return t


t0 = time.perf_counter()
t = t0
x = P.DenseTensor(dims, host).to_device()
t = mark("H2D (to_device)", t)
cfg = P.RunConfig(rank=R, algorithm="hals", max_iters=steps, tol=0.0)
eng = D._Engine(x.data, dims, dims, cfg, D.IdentityCollectives(), None, timing=True, warn_negative=True)
t = mark("engine (alloc + slicing)", t)
eng.initialise()
t = mark("initialise (norm, init err)", t)
eng.iterate()
t = mark(f"{steps} iterations", t)
print("per-iteration wall (ms):", [round(1e3 * w, 1) for w in eng.report.row_wall], "graph:", eng.graph is not None)
owned, lam = eng.model_host()
t = mark("model D2H", t)
print(f"{'total':28s} {1e3 * (t - t0):9.1f} ms  ({8 * host.numel() / 1e9:.1f} GB tensor)")
