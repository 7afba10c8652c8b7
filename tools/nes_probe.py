"""Where do NES traces leave the reference?  Runs the golden NES cases (tests/golden/stateful.npz)
through this package on the GPU and through the UNMODIFIED reference (baseline/_ref) on the host,
logging per outer iteration: the error, every inner-loop step count (mode by mode) with the
stopping quantities, and the outer extrapolation's candidate error vs the current one.

    python tools/nes_probe.py [run-name ...]
"""
import os
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import nncp as R  # noqa: E402  (the reference)
from nncp import driver as RD, updaters as RU  # noqa: E402

import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import driver as PD, updaters as PU  # noqa: E402


def ref_run(x, dims, r, iters, seed):
    log = {"inner": [], "cand": []}
    orig_upd, orig_err = RU.nesterov_update, RD._model_error

    def upd(inp, state, hook=RU.local_reduce, **kw):
        seen = []

        def h(v, op):
            out = hook(v, op)
            seen.append(tuple(np.asarray(out).tolist()))
            return out
        out = orig_upd(inp, state, h, **kw)
        log["inner"].append((state.last_inner_iters, seen[-1]))
        return out

    def merr(*a, **kw):
        e = orig_err(*a, **kw)
        log["cand"].append(e)
        return e
    RU.nesterov_update, RD._model_error = upd, merr
    RD.nesterov_update = upd
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = R.nncp_sequential(R.DenseTensor(dims, x), R.RunConfig(rank=r, algorithm="nes", max_iters=iters,
                                                                        tol=0.0, seed=seed))
    finally:
        RU.nesterov_update, RD._model_error = orig_upd, orig_err
        RD.nesterov_update = orig_upd
    return np.array(rep.errors), log


def our_run(x, dims, r, iters, seed):
    log = {"inner": [], "cand": []}
    orig_run, orig_err = PU.NesterovRunner.run, PD._Engine._model_error

    def run(self, spack, m, current, xstar, hook, *a, **kw):
        seen = []

        def h(v, op):
            out = hook(v, op)
            seen.append(tuple(np.asarray(out.detach().cpu() if hasattr(out, "detach") else out).tolist()))
            return out
        xo, steps = orig_run(self, spack, m, current, xstar, h, *a, **kw)
        log["inner"].append((steps, seen[-1]))
        return xo, steps

    def merr(self, *a):
        e = orig_err(self, *a)
        log["cand"].append(e)
        return e
    PU.NesterovRunner.run, PD._Engine._model_error = run, merr
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=r, algorithm="nes", max_iters=iters,
                                                                        tol=0.0, seed=seed))
    finally:
        PU.NesterovRunner.run, PD._Engine._model_error = orig_run, orig_err
    return np.array(rep.errors), log


def main(names):
    g = np.load(os.path.join(ROOT, "tests", "golden", "stateful.npz"))
    runs = [str(n) for n in g["runs"] if str(g[f"{n}_algo"]) == "nes"]
    for name in names or runs:
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, seed = (int(v) for v in g[f"{name}_meta"])
        x = g[f"{name}_x"]
        re, rl = ref_run(x, dims, r, iters, seed)
        oe, ol = our_run(x, dims, r, iters, seed)
        print(f"== {name} dims={dims} R={r} iters={iters}: max |trace diff| {np.max(np.abs(re - oe)):.3e}, "
              f"ref vs golden {np.max(np.abs(re - g[f'{name}_errors'])):.1e}")
        for it in range(iters):
            print(f"  it {it:2d} eps ref {re[it]:.15e} ours {oe[it]:.15e} diff {oe[it] - re[it]:+.2e}")
        n = len(dims)
        for k, (a, b) in enumerate(zip(rl["inner"], ol["inner"])):
            flag = "" if a[0] == b[0] else "   <-- step count differs"
            print(f"  call {k:3d} (it {k // n}, mode {k % n}) steps ref {a[0]:4d} ours {b[0]:4d}  "
                  f"ref dmax/xmax {a[1][0]:.6e}/{a[1][1]:.6e}  ours {b[1][0]:.6e}/{b[1][1]:.6e}{flag}")
        for k, (a, b) in enumerate(zip(rl["cand"], ol["cand"])):
            print(f"  model_error call {k:3d}: ref {a:.15e} ours {b:.15e} diff {b - a:+.2e}")


if __name__ == "__main__":
    main(sys.argv[1:])
