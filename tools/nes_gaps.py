"""Measured NES trace gaps of every NES comparison the GPU tests make (stateful golden runs,
their (2,2,1) thread-grid runs, runs.npz with the sliced engine forced, sequential vs grid on
uneven blocks), to set the tolerances from data.   python tools/nes_gaps.py"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1909_01149_b200 as P  # noqa: E402

warnings.simplefilter("ignore")
g = np.load(os.path.join(ROOT, "tests", "golden", "stateful.npz"))
for name in [str(n) for n in g["runs"]]:
    algo = str(g[f"{name}_algo"])
    dims = tuple(int(d) for d in g[f"{name}_dims"])
    r, iters, seed = (int(v) for v in g[f"{name}_meta"])
    x = P.DenseTensor(dims, g[f"{name}_x"])
    cfg = dict(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=seed)
    seq = P.nncp_sequential(x, P.RunConfig(**cfg))
    line = f"stateful {name:8s} {algo:4s} seq {np.max(np.abs(np.array(seq.errors) - g[f'{name}_errors'])):.2e}"
    fac = max(np.max(np.abs(seq.model.factors[n] - g[f"{name}_f{n}"])) for n in range(len(dims)))
    line += f" factors {fac:.2e}"
    if f"{name}_grid_errors" in g:
        par = P.nncp_parallel(x, P.RunConfig(**cfg, grid=(2, 2, 1)))
        line += f"  grid {np.max(np.abs(np.array(par.errors) - g[f'{name}_grid_errors'])):.2e}"
    print(line, flush=True)
g = np.load(os.path.join(ROOT, "tests", "golden", "runs.npz"))
for name in [str(n) for n in g["names"]]:
    algo = str(g[f"{name}_algo"])
    if algo != "nes":
        continue
    dims = tuple(int(d) for d in g[f"{name}_dims"])
    r, iters, seed = (int(v) for v in g[f"{name}_meta"])
    x = P.DenseTensor(dims, g[f"{name}_x"])
    for eng in ("sliced", "fp64"):
        rep = P.nncp_sequential(x, P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=seed,
                                               mttkrp_kernel=eng))
        k = min(11, len(g[f"{name}_errors"]))
        d = np.max(np.abs(np.array(rep.errors)[:k] - g[f"{name}_errors"][:k]))
        fac = max(np.max(np.abs(rep.model.factors[n] - g[f"{name}_f{n}"])) for n in range(len(dims)))
        print(f"runs {name:10s} {eng:6s} trace {d:.2e} factors {fac:.2e}", flush=True)
x, _ = P.generate_synthetic(P.SyntheticSpec((7, 5, 6), 2, seed=12))
for algo in ("nes", "admm", "ucp"):
    seq = P.nncp_sequential(x, P.RunConfig(rank=2, algorithm=algo, max_iters=6, tol=0.0, seed=5))
    par = P.nncp_parallel(x, P.RunConfig(rank=2, algorithm=algo, max_iters=6, tol=0.0, seed=5, grid=(2, 2, 1)))
    fac = max(np.max(np.abs(a - b)) for a, b in zip(seq.model.factors, par.model.factors))
    print(f"uneven {algo} seq-vs-grid trace {np.max(np.abs(np.array(seq.errors) - par.errors)):.2e} factors {fac:.2e}")
