"""Randomised parity sweep on the GPU: random shapes, ranks, update rules and
engines against the oracle (sequential) and against the sequential device run
(thread-simulated grids).  Bug hunting beyond the fixed test cases.

    python tools/fuzz_parity.py [cases] [seed] [log2 max elements] [--large]
"""
import sys
import traceback
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from oracle import nncp_oracle as O  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cases = int(args[0]) if len(args) > 0 else 60
rng = np.random.default_rng(int(args[1]) if len(args) > 1 else 7)
warnings.simplefilter("ignore")
LARGE = "--large" in sys.argv
fails = 0
for case in range(cases):
    if LARGE:   # 2^22..2^24 elements: the sizes where "auto" picks the sliced engine
        order = int(rng.integers(3, 5))
        target = 2.0 ** float(rng.uniform(22, 24))
        w = rng.dirichlet(np.ones(order))
        dims = tuple(max(2, int(round(target ** wi))) for wi in w)
    else:
        order = int(rng.integers(2, 6))
        budget = 1 << int(rng.integers(10, int(args[2]) if len(args) > 2 else 19))
        dims = []
        for _ in range(order):
            dims.append(int(rng.integers(1, 48)))
        while np.prod(dims) > budget:
            k = int(np.argmax(dims))
            dims[k] = max(1, dims[k] // 2)
        dims = tuple(dims)
    rank = int(rng.choice([1, 2, 3, 7, 8, 16, 17, 31, 32, 33, 40, 64]))
    algo = str(rng.choice(["mu", "hals", "bpp", "ucp", "admm", "nes"]))
    if LARGE:
        rank = int(rng.choice([8, 16, 20, 32, 33, 48, 64]))
        algo = str(rng.choice(["mu", "hals", "bpp"]))
    engine = str(rng.choice(["fp64", "sliced", "auto"]))
    signed = bool(rng.random() < 0.15) and algo in ("ucp",)
    iters = 4
    hs = [rng.random((d, rank)) for d in dims]
    x = O.khatri_rao(hs) @ np.ones(rank)
    x = x + 0.05 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))
    if signed:
        x = x - np.mean(x)
    scale = 0
    if rng.random() < 0.1:
        scale = int(rng.integers(-60, 60))
        x = x * 2.0 ** scale
    seed = int(rng.integers(0, 100))
    extra = dict(mttkrp_levels=int(rng.choice([6, 6, 7])), dimtree_split=str(rng.choice(["auto", "reference"])),
                 strict_split=bool(rng.random() < 0.2), use_dimtree=bool(rng.random() < 0.85),
                 cuda_graph=[None, False][int(rng.random() < 0.3)])
    tag = f"case {case}: dims {dims} R={rank} {algo} {engine} {extra}" + (f" x*2^{scale}" if scale else "")
    try:
        try:
            ref = O.run_sequential(x, dims, rank, algo, iters, 0.0, seed, use_dimtree=extra["use_dimtree"],
                                   strict_split=extra["strict_split"])
        except Exception as exc:  # noqa: BLE001  (the reference fails too: device must fail alike)
            ref = exc
        try:
            rep = P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=rank, algorithm=algo, max_iters=iters,
                                                                        tol=0.0, seed=seed, mttkrp_kernel=engine, **extra))
        except Exception as exc:  # noqa: BLE001
            if isinstance(ref, Exception):
                print(f"{tag}: both fail ({type(ref).__name__} / {type(exc).__name__})", flush=True)
                continue
            raise
        if isinstance(ref, Exception):
            print(f"{tag}: oracle raised {ref!r}, device did not", flush=True)
            fails += 1
            continue
        errors, factors, lam, _, _ = ref
        tol = 5e-8 if algo == "nes" else 1e-9
        if len(rep.errors) != len(errors):
            # exact fit: eps = sqrt(max(0, radicand)) hits 0 <= tol on one side only
            n = min(len(rep.errors), len(errors))
            tail = max(rep.errors[n - 1], errors[n - 1])
            ok = np.allclose(rep.errors[:n], errors[:n], rtol=0, atol=max(tol, 1e-7)) and tail < 1e-6
            print(f"{tag}: exact fit, traces stop at {len(rep.errors)} / {len(errors)} (eps {tail:.1e})"
                  f"{'' if ok else '  <-- FAIL'}", flush=True)
            fails += 0 if ok else 1
            continue
        # traces compared relative to max(1, eps): a tensor scaled by 2^-60 starts at eps ~ 1e15
        dt = float(np.max(np.abs(np.array(rep.errors) - np.array(errors)) / np.maximum(1.0, np.abs(errors))))
        df = max(float(np.max(np.abs(a - b))) for a, b in zip(rep.model.factors, factors))
        keep = np.abs(lam) > 0
        dl = float(np.max(np.abs(rep.model.lam[keep] - lam[keep]) / np.abs(lam[keep]))) if keep.any() else 0.0
        bad = dt > tol or df > 1e-6 or dl > 1e-6
        grid_msg = ""
        if order >= 2 and rng.random() < 0.5:
            grid = tuple(int(rng.integers(1, min(d, 3) + 1)) for d in dims)
            if np.prod(grid) > 1:
                par = P.nncp_parallel(P.DenseTensor(dims, x), P.RunConfig(rank=rank, algorithm=algo, max_iters=iters,
                                                                           tol=0.0, seed=seed, grid=grid,
                                                                           mttkrp_kernel=engine, **extra))
                if len(par.errors) != len(errors):
                    print(f"{tag}: grid {grid} exact fit, traces stop at {len(par.errors)} / {len(errors)}", flush=True)
                    continue
                dg = float(np.max(np.abs(np.array(par.errors) - np.array(errors)) / np.maximum(1.0, np.abs(errors))))
                dgf = max(float(np.max(np.abs(a - b))) for a, b in zip(par.model.factors, factors))
                grid_msg = f" grid {grid}: trace {dg:.1e} factors {dgf:.1e}"
                bad = bad or dg > tol or dgf > 1e-6
        if bad:
            fails += 1
            print(f"  device {np.array(rep.errors)}\n  oracle {np.array(errors)}", flush=True)
        print(f"{tag}: trace {dt:.1e} factors {df:.1e} lambda {dl:.1e}{grid_msg}{'  <-- FAIL' if bad else ''}", flush=True)
    except Exception:  # noqa: BLE001
        fails += 1
        print(f"{tag}: EXCEPTION\n{traceback.format_exc()}", flush=True)
print(f"{fails} of {cases} cases failed")
