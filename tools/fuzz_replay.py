"""Re-create one case of a tools/fuzz_parity.py log on the CPU and ask whether the
reference itself is rounding-sensitive there (CPU only; needs baseline/_ref or
/root/reference).

    python tools/fuzz_replay.py profiles/r02_fuzz_small_seed2027.log 2027 281
    python tools/fuzz_replay.py profiles/r02_fuzz_large_seed2028.log 2028 27 --large

The fuzz generator's RNG stream depends on which branch each earlier case took (exact
fits and failures skip the grid draws), so the log is read to replay it.  For the case
it prints the UNMODIFIED reference's trace, the change of that trace and of its
factors when the tensor is perturbed by +-1 ulp per element, and the change of the
oracle's trace when only its Gram is summed in 16/32/128-row blocks.
"""
import os
import re
import sys
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "nncp")):
        sys.path.insert(0, cand)
        break
import nncp  # noqa: E402

from oracle import nncp_oracle as O  # noqa: E402


def replay(log, seed, want, large):
    """tools/fuzz_parity.py's draws, case by case, up to case ``want``."""
    lines = {}
    for ln in open(log):
        m = re.match(r"case (\d+): ", ln)
        if m:
            lines[int(m.group(1))] = ln
    rng = np.random.default_rng(seed)
    for case in range(want + 1):
        if large:
            order = int(rng.integers(3, 5))
            target = 2.0 ** float(rng.uniform(22, 24))
            w = rng.dirichlet(np.ones(order))
            dims = tuple(max(2, int(round(target ** wi))) for wi in w)
        else:
            order = int(rng.integers(2, 6))
            budget = 1 << int(rng.integers(10, 19))
            dims = [int(rng.integers(1, 48)) for _ in range(order)]
            while np.prod(dims) > budget:
                k = int(np.argmax(dims))
                dims[k] = max(1, dims[k] // 2)
            dims = tuple(dims)
        rank = int(rng.choice([1, 2, 3, 7, 8, 16, 17, 31, 32, 33, 40, 64]))
        algo = str(rng.choice(["mu", "hals", "bpp", "ucp", "admm", "nes"]))
        if large:
            rank = int(rng.choice([8, 16, 20, 32, 33, 48, 64]))
            algo = str(rng.choice(["mu", "hals", "bpp"]))
        rng.choice(["fp64", "sliced", "auto"])
        signed = bool(rng.random() < 0.15) and algo in ("ucp",)
        hs = [rng.random((d, rank)) for d in dims]
        x = O.khatri_rao(hs) @ np.ones(rank)
        x = x + 0.05 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))
        if signed:
            x = x - np.mean(x)
        if rng.random() < 0.1:
            x = x * 2.0 ** int(rng.integers(-60, 60))
        s = int(rng.integers(0, 100))
        extra = dict(mttkrp_levels=int(rng.choice([6, 6, 7])), dimtree_split=str(rng.choice(["auto", "reference"])),
                     strict_split=bool(rng.random() < 0.2), use_dimtree=bool(rng.random() < 0.85),
                     cuda_graph=[None, False][int(rng.random() < 0.3)])
        ln = lines[case]
        if not ln.startswith(f"case {case}: dims {dims} R={rank} {algo}"):
            raise SystemExit(f"replay diverged at case {case}: {ln.strip()}")
        if case == want:
            return x, dims, rank, algo, s, extra
        seq_fit = " exact fit, traces stop" in ln and "grid (" not in ln.split("exact fit")[0]
        if seq_fit or "both fail" in ln or "oracle raised" in ln:
            continue
        if rng.random() < 0.5:
            tuple(int(rng.integers(1, min(d, 3) + 1)) for d in dims)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    log, seed, case = args[0], int(args[1]), int(args[2])
    x, dims, rank, algo, s, extra = replay(log, seed, case, "--large" in sys.argv)
    warnings.simplefilter("ignore")
    base = dict(rank=rank, algorithm=algo, max_iters=4, tol=0.0, seed=s, strict_split=extra["strict_split"],
                use_dimtree=extra["use_dimtree"])
    ref = nncp.nncp_sequential(nncp.DenseTensor(dims, x), nncp.RunConfig(**base))
    e0 = np.array(ref.errors)
    print(f"case {case}: dims {dims} R={rank} {algo} seed {s}: reference trace {e0}")
    rng = np.random.default_rng(0)
    for k in range(3):
        xp = x * (1 + 2.0 ** -52 * rng.choice([-1, 1], x.size))
        r1 = nncp.nncp_sequential(nncp.DenseTensor(dims, xp), nncp.RunConfig(**base))
        e1 = np.array(r1.errors)
        n = min(len(e0), len(e1))
        dt = float(np.max(np.abs(e1[:n] - e0[:n]) / np.maximum(1.0, e0[:n])))
        df = max(float(np.max(np.abs(a - b))) for a, b in zip(ref.model.factors, r1.model.factors))
        print(f"  reference, tensor * (1 +- 1 ulp) #{k}: trace diff {dt:.2e} (length {len(e1)} vs {len(e0)}), "
              f"factor diff {df:.2e}")
    stock = O.gram
    o = np.array(O.run_sequential(x, dims, rank, algo, 4, 0.0, s, use_dimtree=extra["use_dimtree"],
                                  strict_split=extra["strict_split"])[0])
    for blk in (16, 32, 128):
        def gram(h, blk=blk):
            g = np.zeros((h.shape[1], h.shape[1]))
            for i in range(0, h.shape[0], blk):
                g = g + h[i:i + blk].T @ h[i:i + blk]
            return 0.5 * (g + g.T)
        O.gram = gram
        try:
            a = np.array(O.run_sequential(x, dims, rank, algo, 4, 0.0, s, use_dimtree=extra["use_dimtree"],
                                          strict_split=extra["strict_split"])[0])
        finally:
            O.gram = stock
        n = min(len(a), len(o))
        print(f"  oracle, Gram in {blk}-row blocks: trace diff "
              f"{float(np.max(np.abs(a[:n] - o[:n]) / np.maximum(1.0, o[:n]))):.2e}")


if __name__ == "__main__":
    main()
