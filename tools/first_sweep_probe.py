"""Where the host time of an end-to-end call goes outside the steady sweeps: cProfile of
the engine set-up (slicing included), initialise() and the first (eager) sweep after a
pinned-host H2D, with torch's cudaMalloc count per phase.

    python tools/first_sweep_probe.py 2048x2048x2048 32
"""
import cProfile
import io
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import driver as D  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
R = int(sys.argv[2])
fs = truth_factors(dims, R, 1, "uniform")
xd = synthetic_block(dims, fs, 0.01, 1)
host = torch.empty(xd.numel(), dtype=torch.float64, pin_memory=True)
host.copy_(xd)
del xd
torch.cuda.empty_cache()
torch.cuda.synchronize()


def mallocs():
    return torch.cuda.memory_stats().get("segment.all.allocated", 0)


def phase(label, fn):
    m0 = mallocs()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    out = fn()
    pr.disable()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"== {label}: host {1e3 * (t1 - t0):.1f} ms, + wait for GPU {1e3 * (t2 - t1):.1f} ms, "
          f"cudaMalloc segments +{mallocs() - m0}", flush=True)
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(18)
    print("\n".join(s.getvalue().splitlines()[:40]), flush=True)
    return out


cfg = P.RunConfig(rank=R, algorithm="hals", max_iters=6, tol=0.0)
x = P.DenseTensor(dims, host)
xd = phase("reserve + to_device (async H2D)", lambda: (D._reserve_sliced(dims, cfg), x.to_device())[1])
eng = phase("engine (alloc + slicing)", lambda: D._Engine(xd.data, dims, dims, cfg, D.IdentityCollectives(), None,
                                                           timing=False, warn_negative=True))
phase("initialise", eng.initialise)
phase("sweep 1 (eager)", lambda: eng.iterate(1))
phase("sweep 2 (capture + replay)", lambda: eng.iterate(1))
phase("sweeps 3-6", lambda: eng.iterate(4))
print("row_wall ms:", [round(1e3 * w, 1) for w in eng.report.row_wall])
