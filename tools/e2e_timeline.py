"""Host / GPU timeline of one end-to-end call, as bench.py's e2e leg runs it (stream pool
already built, caches emptied): host timestamps and CUDA events at the phase
boundaries of nncp_sequential, no extra synchronisation between them.

    [E2E_REPS=n] python tools/e2e_timeline.py 2048x2048x2048 32 20
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import driver as D  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
R = int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
torch.cuda.Stream()          # the bench's process has built torch's stream pool already
fs = truth_factors(dims, R, 1, "uniform")
xd = synthetic_block(dims, fs, 0.01, 1)
host = torch.empty(xd.numel(), dtype=torch.float64, pin_memory=True)
host.copy_(xd)
del xd
torch.cuda.empty_cache()
torch.cuda.synchronize()

import os  # noqa: E402

for rep in range(int(os.environ.get("E2E_REPS", "1"))):
    print(f"-- run {rep}")
    marks = []

    def mark(label):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((label, time.perf_counter(), e))

    cfg = P.RunConfig(rank=R, algorithm="hals", max_iters=steps, tol=0.0)
    x = P.DenseTensor(dims, host)
    mark("start")
    D._reserve_sliced(dims, cfg)
    mark("reserved sliced buffer")
    xdev = x.to_device()
    mark("H2D queued")
    eng = D._Engine(xdev.data, dims, dims, cfg, D.IdentityCollectives(), None, timing=False, warn_negative=True)
    mark("engine built (slicing queued)")
    eng.initialise()
    mark("initialised")
    eng.iterate(1)
    mark("sweep 1 (eager)")
    eng.iterate(1)
    mark("sweep 2 (graphs captured)")
    eng.iterate()
    mark(f"sweeps 3-{steps}")
    owned, lam = eng.model_host()
    mark("model D2H")
    torch.cuda.synchronize()
    t0, e0 = marks[0][1], marks[0][2]
    print(f"{'phase end':30s} {'host ms':>9s} {'GPU ms':>9s}")
    for label, t, e in marks:
        print(f"{label:30s} {1e3 * (t - t0):9.1f} {e0.elapsed_time(e):9.1f}")
    del eng, xdev, x
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
