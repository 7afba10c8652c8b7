"""Re-run one tools/fuzz_parity.py case on the GPU with its traces printed in full: the
oracle, the unmodified reference, and the device under engine / graph variants.

    python tools/case_probe.py profiles/r02_fuzz_small_seed2031.log 2031 214
"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from fuzz_replay import nncp, replay  # noqa: E402

from oracle import nncp_oracle as O  # noqa: E402


def main():
    log, seed, case = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    x, dims, rank, algo, s, extra = replay(log, seed, case, "--large" in sys.argv)
    iters = 4
    np.set_printoptions(precision=12, linewidth=160)
    print(f"case {case}: dims {dims} R={rank} {algo} seed {s} {extra}")
    print(f"  x: min {x.min():.3e} max {x.max():.3e} norm {np.linalg.norm(x):.3e}")
    errors = O.run_sequential(x, dims, rank, algo, iters, 0.0, s, use_dimtree=extra["use_dimtree"],
                              strict_split=extra["strict_split"])[0]
    print("  oracle   ", np.array(errors))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        rep = nncp.nncp_sequential(nncp.DenseTensor(dims, x.copy()),
                                   nncp.RunConfig(rank=rank, algorithm=algo, max_iters=iters, tol=0.0, seed=s,
                                                  use_dimtree=extra["use_dimtree"],
                                                  strict_split=extra["strict_split"]))
    print("  reference", np.array(rep.errors))
    import paper_1909_01149_b200 as P

    for engine in ("auto", "fp64"):
        for graph in (None, False):
            cfg = dict(extra, cuda_graph=graph)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                r = P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=rank, algorithm=algo, max_iters=iters,
                                                                          tol=0.0, seed=s, mttkrp_kernel=engine, **cfg))
            print(f"  device {engine:5s} graph={graph!s:5s}", np.array(r.errors), " lam", r.model.lam[:4])
    for grid in [(3, 1), (1, 1), (2, 1)]:
        if len(grid) != len(dims):
            continue
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = P.nncp_parallel(P.DenseTensor(dims, x), P.RunConfig(rank=rank, algorithm=algo, max_iters=iters,
                                                                    tol=0.0, seed=s, grid=grid, **extra))
        print(f"  device grid {grid}", np.array(r.errors))


if __name__ == "__main__":
    main()
