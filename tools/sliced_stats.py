"""Barrier wait-cycle breakdown of the sliced GEMM (instrumented build).

    python -m paper_1909_01149_b200.build_ext --stats
    NNCP_LIB_PATH=paper_1909_01149_b200/libnncp_b200_stats.so python tools/sliced_stats.py 2048x2048x2048:64
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import _lib, synth  # noqa: E402
from paper_1909_01149_b200.dimtree import SlicedTensor  # noqa: E402

lib = _lib.load()
fn = lib.nncp_sliced_stats
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.c_int]
buf = (ctypes.c_ulonglong * (1024 * 8))()
SUSTAIN = int(__import__("os").environ.get("SUSTAIN", "1"))
names = ["prod:B empty", "prod:A empty", "mma:TMEM empty", "mma:B full", "mma:A full", "epi:TMEM full", "kernel"]
for spec in sys.argv[1:]:
    dims_s, r_s = spec.split(":")
    dims = tuple(int(d) for d in dims_s.split("x"))
    r = int(r_s)
    x = synth.synthetic_block(dims, synth.truth_factors(dims, r, 1, "uniform"), 0.01, 1)
    plan = P.DimTreePlan.create(dims, r)
    sl = SlicedTensor(x, dims, plan.split)
    hs = [torch.rand(d, r, dtype=torch.float64, device="cuda") for d in dims]
    ws = P.tensor_ops.Workspace(max(plan.workspace_bytes(), plan.sliced_workspace_bytes()))
    for side in ("left", "right"):
        # sustained: back-to-back calls first, so the measured one runs at the power-capped clock
        for _ in range(SUSTAIN):
            P.partial_mttkrp(x, hs, side, plan, workspace=ws, sliced=sl)
        torch.cuda.synchronize()
        fn(buf, 1024 * 8, 1)
        P.partial_mttkrp(x, hs, side, plan, workspace=ws, sliced=sl)
        torch.cuda.synchronize()
        fn(buf, 1024 * 8, 1)
        a = np.array(buf[:148 * 8], dtype=np.float64).reshape(148, 8)
        used = a[:, 6] > 0
        k = a[used].mean(axis=0)
        k[5] /= 256.0   # every thread of the 8 epilogue warps adds its own wait
        print(f"{spec} {side}: kernel {k[6] / 1e3:.1f} kcycles/CTA; waits (% of kernel cycles): "
              + ", ".join(f"{n} {100 * k[i] / k[6]:.1f}" for i, n in enumerate(names[:6])), flush=True)
    del sl, x, ws
    torch.cuda.empty_cache()
