"""Run the two partial MTTKRP kernels on a synthetic tensor (for ncu / quick timing).

    python tools/profile_partial.py --dims 2048,2048,512 --rank 32 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402
from paper_1909_01149_b200.tensor_ops import Workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="2048,2048,512")
ap.add_argument("--rank", type=int, default=32)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sides", default="left,right")
a = ap.parse_args()
dims = tuple(int(v) for v in a.dims.split(","))
fs = truth_factors(dims, a.rank, 1)
x = synthetic_block(dims, fs, 0.01, 1)
plan = P.DimTreePlan.create(dims, a.rank)
ws = Workspace(plan.workspace_bytes())
hs = [torch.from_numpy(f).cuda() for f in fs]
size = int(np.prod(dims))
for side in a.sides.split(","):
    out = None
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t = P.partial_mttkrp(x, hs, side, plan, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        out = t.data
        times.append(e0.elapsed_time(e1) / 1e3)
    best = min(times)
    print(f"{side}: {best * 1e3:.3f} ms  {2 * size * a.rank / best / 1e12:.2f} TFLOP/s  "
          f"{8 * size / best / 1e9:.0f} GB/s")
