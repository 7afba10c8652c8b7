"""Sliced partial MTTKRP timing in three settings, to separate kernel time from what the
surrounding sweep adds: (1) each call alone (sync before/after), (2) back-to-back calls,
(3) back-to-back calls replayed from a CUDA graph, each preceded by a 2 MB fill (a
small-kernel stand-in, as in the sweep).

    python tools/partial_ingraph.py 1024x1024x1024 32
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200.dimtree import SlicedTensor  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402
from paper_1909_01149_b200.tensor_ops import Workspace  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
R = int(sys.argv[2])
reps = 10
fs = truth_factors(dims, R, 1, "uniform")
x = synthetic_block(dims, fs, 0.01, 1)
plan = P.DimTreePlan.create(dims, R)
sl = SlicedTensor(x, dims, plan.split, 6)
ws = Workspace(plan.sliced_workspace_bytes(6))
hs = [torch.from_numpy(f).cuda() for f in fs]
outs = {s: torch.empty(int(np.prod(dims[:plan.split] if s == "left" else dims[plan.split:])) * R,
                       dtype=torch.float64, device="cuda") for s in ("left", "right")}
scratch = torch.empty(1 << 18, dtype=torch.float64, device="cuda")


def call(side):
    P.partial_mttkrp(x, hs, side, plan, out=outs[side], workspace=ws, sliced=sl)


def ev():
    return torch.cuda.Event(enable_timing=True)


for side in ("left", "right"):
    call(side)
torch.cuda.synchronize()
for side in ("left", "right"):
    alone = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        call(side)
        b.record()
        torch.cuda.synchronize()
        alone.append(a.elapsed_time(b))
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        call(side)
    b.record()
    torch.cuda.synchronize()
    b2b = a.elapsed_time(b) / reps
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin()
        for _ in range(reps):
            scratch.fill_(1.0)
            call(side)
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    gr = a.elapsed_time(b) / reps
    print(f"{side}: alone min {min(alone):.3f} median {np.median(alone):.3f} ms | back-to-back {b2b:.3f} | "
          f"graph (with a 2 MB fill before each) {gr:.3f} ms", flush=True)
