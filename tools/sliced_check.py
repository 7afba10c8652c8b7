"""Sliced (int8 tensor-core) vs FP64 DMMA partial MTTKRPs at large shapes: error and timing."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import synth  # noqa: E402
from paper_1909_01149_b200.dimtree import SlicedTensor  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for spec in sys.argv[1:]:
    dims_s, r_s = spec.split(":")
    dims = tuple(int(d) for d in dims_s.split("x"))
    r = int(r_s)
    fs = synth.truth_factors(dims, r, 1, "uniform")
    x = synth.synthetic_block(dims, fs, 0.01, 1)
    plan = P.DimTreePlan.create(dims, r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sl = SlicedTensor(x, dims, plan.split)
    torch.cuda.synchronize()
    t_slice = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    hs = [torch.from_numpy(rng.random((d, r))).cuda() for d in dims]
    ws = P.tensor_ops.Workspace(max(plan.workspace_bytes(), plan.sliced_workspace_bytes()))
    for side in ("left", "right"):
        ref = P.partial_mttkrp(x, hs, side, plan, workspace=ws).data.clone()
        got = P.partial_mttkrp(x, hs, side, plan, workspace=ws, sliced=sl).data.clone()
        err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
        bad = torch.nonzero(~torch.isclose(got, ref, rtol=1e-10, atol=0))
        t64 = timed(lambda: P.partial_mttkrp(x, hs, side, plan, workspace=ws))
        t8 = timed(lambda: P.partial_mttkrp(x, hs, side, plan, workspace=ws, sliced=sl))
        nel = int(np.prod(dims))
        print(f"{spec} {side}: rel_err {err:.3e} bad {bad.shape[0]} first {bad[:4].flatten().tolist()} "
              f"fp64 {t64:.3f} ms sliced {t8:.3f} ms ({6 * nel / t8 / 1e6:.0f} GB/s of planes) slice-once {t_slice*1e3:.1f} ms",
              flush=True)
    del sl, x, ws
    torch.cuda.empty_cache()
