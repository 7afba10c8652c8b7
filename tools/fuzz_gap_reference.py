"""The two fuzz mismatches of round 1 (tensors scaled by 2^-57 / 2^-51 against U[0,1)
initial factors) re-run on the UNMODIFIED reference itself: its own sequential and
grid runs disagree by the same order, i.e. the inputs are ill-posed, not the device
path wrong.  CPU only; needs /root/reference (or baseline/_ref).

    python tools/fuzz_gap_reference.py > profiles/r02_fuzz_gap_reference.log
"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "nncp")):
        sys.path.insert(0, cand)
        break
import nncp  # noqa: E402

warnings.simplefilter("ignore")
CASES = [((4, 5, 4, 6), 40, "hals", -57, (3, 1, 2, 3), True),      # round-1 fuzz9 case 77
         ((1347, 6, 11, 102), 64, "hals", -51, (3, 1, 1, 1), False)]  # round-1 fuzz12 case 9
for dims, rank, algo, scale, grid, strict in CASES:
    for seed in range(3):
        rng = np.random.default_rng(seed)
        hs = [rng.random((d, rank)) for d in dims]
        x = nncp.khatri_rao(hs) @ np.ones(rank)
        x = (x + 0.05 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))) * 2.0 ** scale
        t = nncp.DenseTensor(dims, x)
        cfg = dict(rank=rank, algorithm=algo, max_iters=4, tol=0.0, seed=seed, strict_split=strict)
        seq = np.array(nncp.nncp_sequential(t, nncp.RunConfig(**cfg)).errors)
        par = np.array(nncp.nncp_parallel(t, nncp.RunConfig(grid=grid, **cfg)).errors)
        # unscaled control: the same data at scale 2^0
        t1 = nncp.DenseTensor(dims, x * 2.0 ** -scale)
        seq1 = np.array(nncp.nncp_sequential(t1, nncp.RunConfig(**cfg)).errors)
        par1 = np.array(nncp.nncp_parallel(t1, nncp.RunConfig(grid=grid, **cfg)).errors)
        print(f"dims {dims} R={rank} {algo} x*2^{scale} grid {grid} seed {seed}: reference seq vs grid trace diff "
              f"{np.max(np.abs(seq - par) / np.maximum(1.0, seq)):.2e}   (unscaled control: "
              f"{np.max(np.abs(seq1 - par1)):.2e});  eps[0..] {seq[:3]}")
