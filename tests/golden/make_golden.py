"""Generate golden fixtures by running the LIVE reference package.

Run in the build container only (the reference tree does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array in the resulting ``tests/golden/*.npz`` files is an input we
chose (seeded numpy draws) or an output computed by the unmodified
reference (`nncp` package: dimtree.py, updaters.py, driver.py).  The tests
compare both the CPU oracle (``oracle/nncp_oracle.py``) and the CUDA path
against these files.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import nncp  # noqa: E402  (the reference)
from nncp import (  # noqa: E402
    DenseTensor, DimTreeContext, DimTreePlan, FactorSet, RunConfig, UpdateInputs,
    bpp_update, hals_update, khatri_rao, mu_update, naive_mttkrp, nncp_parallel,
    nncp_sequential, partial_mttkrp, multi_ttv,
)

OUT = os.path.dirname(os.path.abspath(__file__))


def noisy_lowrank(rng, dims, rank, eta):
    """Nonneg rank-R tensor from U[0,1) factors plus eta*rms*|N(0,1)| noise."""
    hs = [rng.random((d, rank)) for d in dims]
    clean = khatri_rao(hs) @ np.ones(rank)
    rms = float(np.sqrt(np.mean(clean * clean)))
    return clean + eta * rms * np.abs(rng.standard_normal(clean.size))


def mttkrp_cases():
    """Dimension-tree MTTKRP (all modes, with factor mutation) + last-mode shortcut."""
    rng = np.random.default_rng(2024)
    shapes = [((6, 5, 4), 3), ((7, 5, 6), 2), ((8, 8, 8), 16), ((16, 12, 10), 10),
              ((6, 5, 4, 3), 4), ((4, 6, 5, 3), 20), ((3, 4, 2, 3, 2), 3), ((9, 4), 5),
              ((32, 16, 24), 32), ((10, 8, 6, 4), 64), ((5, 7, 3), 1), ((12, 2, 30), 24)]
    out = {}
    for k, (dims, r) in enumerate(shapes):
        x = DenseTensor(dims, rng.standard_normal(int(np.prod(dims))))
        hs = [rng.standard_normal((d, r)) for d in dims]
        ctx = DimTreeContext(DimTreePlan.create(dims, r))
        ctx.begin_iteration()
        cur = [h.copy() for h in hs]
        res, used = [], []
        for n in range(len(dims)):
            used.append([h.copy() for h in cur])
            res.append(ctx.mttkrp(x, cur, n))
            cur[n] = rng.standard_normal(cur[n].shape)  # the "update"
        last = DimTreeContext(DimTreePlan.create(dims, r)).mttkrp_last_mode(x, hs)
        out[f"c{k}_dims"] = np.array(dims)
        out[f"c{k}_rank"] = np.array(r)
        out[f"c{k}_x"] = x.data
        for n in range(len(dims)):
            out[f"c{k}_h{n}"] = hs[n]
            out[f"c{k}_new{n}"] = cur[n]
            out[f"c{k}_m{n}"] = res[n]
        out[f"c{k}_last"] = last
        out[f"c{k}_split"] = np.array(ctx.plan.split)
        # naive (einsum) oracle for mode N-1 with the original factors
        out[f"c{k}_naive_last"] = naive_mttkrp(x, hs, len(dims) - 1)
        # partial MTTKRPs and TTVs on their own
        plan = ctx.plan
        s = plan.split
        tl = partial_mttkrp(x, khatri_rao(hs[s:]), "left", plan)
        tr = partial_mttkrp(x, khatri_rao(hs[:s]), "right", plan)
        out[f"c{k}_tl"] = tl.data
        out[f"c{k}_tr"] = tr.data
        if s >= 2:
            out[f"c{k}_ttv_trail"] = multi_ttv(tl, khatri_rao(hs[1:s]), "trailing").data
            out[f"c{k}_ttv_lead"] = multi_ttv(tl, hs[0], "leading").data
    out["ncases"] = np.array(len(shapes))
    np.savez_compressed(os.path.join(OUT, "mttkrp.npz"), **out)


def update_cases():
    """MU / HALS / BPP on SPD Grams from nonneg data, various ranks."""
    rng = np.random.default_rng(77)
    out = {}
    k = 0
    for r in (1, 2, 3, 5, 8, 10, 16, 20, 32):
        for rows in (1, 7, 33):
            a = rng.random((r + 6, r))
            b = rng.random((r + 6, rows))
            s = a.T @ a
            s = 0.5 * (s + s.T)
            m = b.T @ a
            # a signed variant makes BPP pivot more
            if k % 2 == 1:
                m = m - 0.6 * np.abs(m).mean()
            cur = rng.random((rows, r)) + 1e-3
            out[f"u{k}_s"], out[f"u{k}_m"], out[f"u{k}_cur"] = s, m, cur
            out[f"u{k}_mu"] = mu_update(UpdateInputs(s, m, cur))
            out[f"u{k}_hals"] = hals_update(UpdateInputs(s, m, cur))
            out[f"u{k}_bpp"] = bpp_update(UpdateInputs(s, m, cur))
            k += 1
    out["nupd"] = np.array(k)
    # HALS zero diagonal (test_updaters.py:124-129) and BPP cycling (193-198)
    out["hals_zero_s"] = np.array([[1.0, 0.0], [0.0, 0.0]])
    out["hals_zero_m"] = np.array([[1.0, 5.0]])
    out["hals_zero_cur"] = np.array([[0.0, 0.25]])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out["hals_zero_out"] = hals_update(
            UpdateInputs(out["hals_zero_s"], out["hals_zero_m"], out["hals_zero_cur"]))
    out["bpp_cycle_s"] = np.array([[1.0, -3.0], [-3.0, 1.0]])
    out["bpp_cycle_m"] = np.array([[0.0, 0.0], [1.0, 1.0]])
    np.savez_compressed(os.path.join(OUT, "updates.npz"), **out)


def run_cases():
    """Full sequential runs (error trace, final model) + grid runs."""
    out = {}
    cases = [
        # name, dims, rank, algo, iters, data seed, init seed, eta
        ("c1_mu", (64, 64, 64), 10, "mu", 20, 1, 0, 0.01),  # BASELINE configs[0]
        ("hals3", (24, 20, 16), 5, "hals", 15, 2, 0, 0.01),
        ("bpp3", (18, 16, 14), 4, "bpp", 12, 3, 1, 0.01),
        ("mu4", (8, 7, 6, 5), 3, "mu", 10, 4, 2, 0.01),
        ("hals4", (10, 9, 8, 7), 6, "hals", 10, 5, 3, 0.02),
        ("bpp4", (9, 8, 7, 6), 5, "bpp", 10, 6, 4, 0.01),
        ("hals_r16", (32, 32, 32), 16, "hals", 10, 7, 0, 0.01),
        ("bpp_r32", (40, 36, 34), 32, "bpp", 6, 8, 0, 0.01),
        ("hals_odd", (7, 5, 6), 2, "hals", 10, 9, 5, 0.05),
        ("mu_2way", (30, 20), 4, "mu", 10, 10, 0, 0.01),
        ("bpp_5way", (4, 5, 3, 4, 3), 2, "bpp", 8, 11, 0, 0.01),
        ("hals_img", (64, 32, 8), 20, "hals", 8, 12, 0, 0.05),
    ]
    for name, dims, r, algo, iters, dseed, iseed, eta in cases:
        rng = np.random.default_rng(1000 + dseed)
        data = noisy_lowrank(rng, dims, r, eta)
        x = DenseTensor(dims, data)
        cfg = RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed)
        rep = nncp_sequential(x, cfg)
        out[f"{name}_dims"] = np.array(dims)
        out[f"{name}_meta"] = np.array([r, iters, iseed])
        out[f"{name}_algo"] = np.array(algo)
        out[f"{name}_x"] = data
        out[f"{name}_errors"] = np.array(rep.errors)
        out[f"{name}_lam"] = rep.model.lam
        out[f"{name}_split"] = np.array(rep.split_mode)
        for n, h in enumerate(rep.model.factors):
            out[f"{name}_f{n}"] = h
    out["names"] = np.array([c[0] for c in cases])
    # grid runs of the reference's simulated-parallel driver
    grids = [("hals_odd", (2, 2, 1)), ("bpp3", (2, 2, 2)), ("mu4", (2, 1, 2, 1)),
             ("hals4", (2, 2, 2, 1)), ("bpp4", (1, 2, 2, 2))]
    for name, grid in grids:
        dims = tuple(out[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in out[f"{name}_meta"])
        algo = str(out[f"{name}_algo"])
        x = DenseTensor(dims, out[f"{name}_x"])
        par = nncp_parallel(x, RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0,
                                         seed=iseed, grid=grid))
        tag = f"grid_{name}_" + "x".join(map(str, grid))
        out[f"{tag}_errors"] = np.array(par.errors)
        out[f"{tag}_split"] = np.array(par.split_mode)
        out[f"{tag}_calls"] = np.array([par.counters.calls.get(c, 0) for c in
                                        ("ReduceScatter", "AllGather", "AllReduce")])
        out[f"{tag}_words_in"] = np.array([par.counters.words_in.get(c, 0) for c in
                                           ("ReduceScatter", "AllGather", "AllReduce")])
        out[f"{tag}_words_out"] = np.array([par.counters.words_out.get(c, 0) for c in
                                            ("ReduceScatter", "AllGather", "AllReduce")])
        for n, h in enumerate(par.model.factors):
            out[f"{tag}_f{n}"] = h
    out["grids"] = np.array([f"grid_{n}_" + "x".join(map(str, g)) for n, g in grids])
    np.savez_compressed(os.path.join(OUT, "runs.npz"), **out)


def init_cases():
    """init_factor draws (driver.py:137-143) for a few (seed, mode, rows, rank)."""
    from nncp import init_factor
    out = {}
    for k, (seed, mode, rows, rank) in enumerate([(0, 0, 5, 3), (3, 1, 10, 4), (7, 2, 12, 3),
                                                    (123456789, 3, 4, 32)]):
        out[f"i{k}_args"] = np.array([seed, mode, rows, rank])
        out[f"i{k}_val"] = init_factor(seed, mode, rows, rank)
    np.savez_compressed(os.path.join(OUT, "init.npz"), **out)


def stateful_cases():
    """UCP / ADMM / NES (updaters.py:77-88,167-281) on the update inputs + full runs."""
    from nncp import UpdaterState, admm_update, nesterov_update, ucp_update
    from nncp.updaters import nesterov_hyperparams

    rng = np.random.default_rng(91)
    out = {}
    k = 0
    for r in (1, 2, 3, 5, 8, 16, 20, 32):
        for rows in (1, 9, 40):
            a = rng.random((r + 6, r))
            b = rng.random((r + 6, rows))
            s = a.T @ a
            s = 0.5 * (s + s.T)
            m = b.T @ a
            if k % 2 == 1:
                m = m - 0.5 * np.abs(m).mean()
            cur = rng.random((rows, r)) + 1e-3
            out[f"s{k}_s"], out[f"s{k}_m"], out[f"s{k}_cur"] = s, m, cur
            out[f"s{k}_ucp"] = ucp_update(UpdateInputs(s, m, cur))
            st = UpdaterState()
            out[f"s{k}_admm1"] = admm_update(UpdateInputs(s, m, cur), st)
            out[f"s{k}_admm1_iters"] = np.array(st.last_inner_iters)
            out[f"s{k}_admm2"] = admm_update(UpdateInputs(s, m, out[f"s{k}_admm1"]), st)
            out[f"s{k}_admm_dual"] = st.admm_dual
            nst = UpdaterState()
            out[f"s{k}_nes"] = nesterov_update(UpdateInputs(s, m, cur), nst)
            out[f"s{k}_nes_iters"] = np.array(nst.last_inner_iters)
            out[f"s{k}_hyper"] = np.array(nesterov_hyperparams(s))
            k += 1
    out["nst"] = np.array(k)
    # runs
    cases = [("ucp3", (12, 10, 8), 3, "ucp", 6, 21), ("admm3", (14, 12, 10), 4, "admm", 8, 22),
             ("nes3", (12, 11, 10), 3, "nes", 8, 23), ("admm4", (7, 6, 5, 4), 3, "admm", 6, 24),
             ("nes4", (7, 6, 5, 4), 2, "nes", 6, 25), ("nes_r16", (24, 20, 18), 16, "nes", 5, 26)]
    for name, dims, r, algo, iters, dseed in cases:
        rng2 = np.random.default_rng(dseed)
        data = noisy_lowrank(rng2, dims, r, 0.02)
        x = DenseTensor(dims, data)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = nncp_sequential(x, RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=1))
        out[f"{name}_dims"] = np.array(dims)
        out[f"{name}_meta"] = np.array([r, iters, 1])
        out[f"{name}_algo"] = np.array(algo)
        out[f"{name}_x"] = data
        out[f"{name}_errors"] = np.array(rep.errors)
        out[f"{name}_lam"] = rep.model.lam
        out[f"{name}_partials"] = np.array(rep.tree_partial_calls)
        for n, h in enumerate(rep.model.factors):
            out[f"{name}_f{n}"] = h
        if name in ("admm3", "nes3"):
            par = nncp_parallel(x, RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=1,
                                             grid=(2, 2, 1)))
            out[f"{name}_grid_errors"] = np.array(par.errors)
            out[f"{name}_grid_calls"] = np.array([par.counters.calls.get(c, 0) for c in
                                                  ("ReduceScatter", "AllGather", "AllReduce")])
    out["runs"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(OUT, "stateful.npz"), **out)


def synthetic_cases():
    """Reference generate_synthetic truth factors + tensor (tensor_io.py:103-125)."""
    from nncp import SyntheticSpec, generate_synthetic

    spec = SyntheticSpec((9, 8, 7), 3, seed=13)
    x, truth = generate_synthetic(spec)
    out = {"dims": np.array(spec.dims), "rank": np.array(spec.rank), "seed": np.array(spec.seed), "x": x.data}
    for n, h in enumerate(truth.factors):
        out[f"h{n}"] = h
    np.savez_compressed(os.path.join(OUT, "synthetic.npz"), **out)


if __name__ == "__main__":
    print("reference nncp", nncp.__version__, "numpy", np.__version__)
    mttkrp_cases()
    update_cases()
    run_cases()
    init_cases()
    synthetic_cases()
    stateful_cases()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


