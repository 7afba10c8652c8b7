"""Full-size c5 parity log: the device run vs the CPU reference on
identical input bits, 10 outer iterations, at 2048^3.

    python tools/c5_parity.py [--rank 32] [--algo hals] [--checker reference|oracle]

The tensor is generated once in HBM (bench.py's seeded generator), the device runs
both MTTKRP engines (default sliced int8 tensor cores; FP64 DMMA), then the tensor is
copied to the host and the checker runs: the UNMODIFIED reference nncp_sequential from
baseline/_ref (its init row is the einsum MTTKRP, ~4 min at this size) or the oracle
port (tests' checker, init error through the tree).  Prints both traces, the per-
iteration differences and the factor / lambda differences against north_star's
tolerances (traces <= 1e-9 over the first 10 iterations, factors <= 1e-6).
"""

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=32)
    ap.add_argument("--algo", default="hals")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--checker", default="reference", choices=["reference", "oracle"])
    args = ap.parse_args()
    import torch

    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200.synth import synthetic_block, truth_factors

    dims = (2048, 2048, 2048)
    fs = truth_factors(dims, args.rank, 1)
    x = synthetic_block(dims, fs, 0.01, 1)
    dev = {}
    for engine in ("sliced", "fp64"):
        t0 = time.perf_counter()
        cfg = P.RunConfig(rank=args.rank, algorithm=args.algo, max_iters=args.iters, tol=0.0, mttkrp_kernel=engine)
        eng, rep = P.run_local(x, dims, dims, cfg)
        f, lam = eng.model_host()
        dev[engine] = (np.array(rep.errors), f, lam, eng.sliced is not None)
        del eng
        torch.cuda.empty_cache()
        print(f"device {engine}: {time.perf_counter() - t0:.1f} s (init + {args.iters} iterations + slicing)",
              flush=True)
    host = x.cpu().numpy()
    del x
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    if args.checker == "reference":
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        import nncp

        ref = nncp.nncp_sequential(nncp.DenseTensor(dims, host),
                                   nncp.RunConfig(rank=args.rank, algorithm=args.algo, max_iters=args.iters, tol=0.0,
                                                  seed=0))
        errors, factors, lam = np.array(ref.errors), ref.model.factors, ref.model.lam
        what = "unmodified reference nncp_sequential (baseline/_ref)"
    else:
        from oracle import nncp_oracle as O

        e, factors, lam, _, _ = O.run_sequential(host, dims, args.rank, args.algo, args.iters, 0.0, 0,
                                                 init_error="tree")
        errors = np.array(e)
        what = "oracle port (init error through the tree)"
    print(f"checker: {what}: {time.perf_counter() - t0:.1f} s", flush=True)
    print(f"c5 {'x'.join(map(str, dims))} R={args.rank} {args.algo.upper()} {args.iters} iterations, seed 0, "
          f"data seed 1, 1% |Gaussian| noise")
    print(f"{'it':>3} {'checker eps':>22} {'sliced eps':>22} {'fp64 eps':>22} {'|sliced-chk|':>12} {'|fp64-chk|':>12}")
    es, ef = dev["sliced"][0], dev["fp64"][0]
    for k in range(len(errors)):
        print(f"{k:>3} {errors[k]:>22.17g} {es[k]:>22.17g} {ef[k]:>22.17g} {abs(es[k] - errors[k]):>12.2e} "
              f"{abs(ef[k] - errors[k]):>12.2e}")
    ok = True
    for engine in ("sliced", "fp64"):
        e, f, lm, sliced = dev[engine]
        trace = float(np.max(np.abs(e[:11] - errors[:11])))
        fac = max(float(np.max(np.abs(a - b))) for a, b in zip(f, factors))
        lrel = float(np.max(np.abs(lm - lam) / np.abs(lam)))
        good = trace <= 1e-9 and fac <= 1e-6
        ok &= good
        print(f"{engine:>6} (sliced engine in use: {sliced}): trace diff {trace:.2e} (tol 1e-9), factor diff "
              f"{fac:.2e} (tol 1e-6), lambda rel diff {lrel:.2e} -> {'PASS' if good else 'FAIL'}")
    print("RESULT", "PASS" if ok else "FAIL")


if __name__ == "__main__":
    main()
