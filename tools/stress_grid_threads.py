"""Repeat a thread-simulated grid run against the sequential run (race hunting)."""
import sys
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "admm"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
x, _ = P.generate_synthetic(P.SyntheticSpec((7, 5, 6), 2, seed=12))
warnings.simplefilter("ignore")
seq = P.nncp_sequential(x, P.RunConfig(rank=2, algorithm=algo, max_iters=6, tol=0.0, seed=5))
bad = 0
for k in range(reps):
    par = P.nncp_parallel(x, P.RunConfig(rank=2, algorithm=algo, max_iters=6, tol=0.0, seed=5, grid=(2, 2, 1)))
    d = float(np.max(np.abs(np.array(seq.errors) - np.array(par.errors))))
    if d > 1e-10:
        bad += 1
        print(f"rep {k}: trace diff {d:.3e}  par {par.errors[:3]}", flush=True)
print(f"{algo}: {bad} of {reps} grid runs differ")
