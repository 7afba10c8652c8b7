"""Sliced-tensor partial MTTKRP (int8 tensor cores, Ozaki-scheme digit planes;
DESIGN.md §4.4) vs the reference's golden vectors, the CPU oracle and the FP64
DMMA path.  Same tolerances as every other MTTKRP in the north star: <= 1e-12
relative Frobenius for a single MTTKRP, error traces <= 1e-9 over the first
10 iterations, final normalised factors <= 1e-6."""

import warnings

import numpy as np
import pytest

from oracle import nncp_oracle as O
from tests.conftest import rel_fro

pytestmark = pytest.mark.gpu

MTTKRP_TOL = 1e-12
TRACE_TOL = 1e-9
FACTOR_TOL = 1e-6


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as pkg

    return pkg


def _np(t):
    """Host copy of a result: device tensors for device inputs, numpy (as the reference) for host inputs."""
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def _sliced(P, x, plan, levels=6):
    from paper_1909_01149_b200.dimtree import SlicedTensor

    return SlicedTensor(x, plan.dims, plan.split, levels)


@pytest.mark.parametrize("levels", [6, 7])
def test_sliced_partials_vs_golden(P, golden, levels):
    g = golden("mttkrp.npz")
    for k in range(int(g["ncases"])):
        dims = tuple(int(d) for d in g[f"c{k}_dims"])
        r = int(g[f"c{k}_rank"])
        x = P.DenseTensor(dims, g[f"c{k}_x"]).to_device()
        hs = [g[f"c{k}_h{n}"] for n in range(len(dims))]
        plan = P.DimTreePlan.create(dims, r)
        sl = _sliced(P, x, plan, levels)
        tl = P.partial_mttkrp(x, hs, "left", plan, sliced=sl)
        tr = P.partial_mttkrp(x, hs, "right", plan, sliced=sl)
        assert rel_fro(_np(tl.data), g[f"c{k}_tl"]) <= MTTKRP_TOL, (k, dims, r)
        assert rel_fro(_np(tr.data), g[f"c{k}_tr"]) <= MTTKRP_TOL, (k, dims, r)


@pytest.mark.parametrize("dims,r", [((128, 96, 80), 32), ((64, 48, 40, 24), 16), ((4096, 64, 32), 20),
                                    ((100, 64, 64), 64), ((256, 256, 300), 8), ((7, 9, 11), 5),
                                    ((96, 64, 48), 40), ((64, 64, 64, 8), 48), ((130, 70, 50), 56),
                                    ((30, 20, 10, 8, 6), 12), ((2, 3, 4, 5, 6, 7), 3), ((33, 17, 5), 1),
                                    ((257, 129, 65), 33)])
def test_sliced_partials_vs_oracle(P, dims, r):
    rng = np.random.default_rng(sum(dims) + r)
    x = rng.random(int(np.prod(dims)))
    hs = [rng.random((d, r)) for d in dims]
    plan = P.DimTreePlan.create(dims, r)
    xd = P.DenseTensor(dims, x).to_device()
    sl = _sliced(P, xd, plan)
    for side, fn in (("left", O.partial_left), ("right", O.partial_right)):
        got = _np(P.partial_mttkrp(xd, hs, side, plan, sliced=sl).data)
        want = fn(x, dims, plan.split, hs)
        assert rel_fro(got, want) <= MTTKRP_TOL, side


@pytest.mark.parametrize("dims,r", [((512, 512, 512), 16), ((180, 100, 17000), 32), ((64, 64, 64, 64), 64),
                                    ((2048, 1024, 60), 20), ((1000, 1000, 999), 48)])
def test_sliced_vs_fp64_path_multichunk(P, dims, r):
    """Shapes with several contraction chunks (K > 16384 on the left, split-K groups on the right),
    uneven tiles, R padded to 16/48/64: sliced == FP64 DMMA path (itself oracle-checked) to 1e-12."""
    import torch

    from paper_1909_01149_b200 import synth

    fs = synth.truth_factors(dims, r, 7, "uniform")
    x = synth.synthetic_block(dims, fs, 0.01, 7)
    plan = P.DimTreePlan.create(dims, r)
    rng = np.random.default_rng(r)
    hs = [torch.from_numpy(rng.random((d, r))).cuda() for d in dims]
    sl = _sliced(P, x, plan)
    for side in ("left", "right"):
        ref = P.partial_mttkrp(x, hs, side, plan).data
        got = P.partial_mttkrp(x, hs, side, plan, sliced=sl).data
        err = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
        assert err <= MTTKRP_TOL, (side, err)
    del sl, x
    torch.cuda.empty_cache()


def test_sliced_signed_and_wide_range(P):
    """Mixed-sign tensors and factors, zeros, and per-row magnitudes over 2^40: the
    row / column-chunk scales keep every row at full relative precision."""
    dims, r = (300, 200, 150), 24
    rng = np.random.default_rng(5)
    x = rng.standard_normal(int(np.prod(dims)))
    rows = np.prod(dims[:2])
    x = x.reshape(dims[2], rows) * np.exp2(rng.integers(-20, 20, rows))[None, :]   # per-row scale (left side rows)
    x[:, ::7] = 0.0
    x = x.ravel()
    hs = [rng.standard_normal((d, r)) for d in dims]
    plan = P.DimTreePlan.create(dims, r)
    xd = P.DenseTensor(dims, x).to_device()
    sl = _sliced(P, xd, plan, 7)
    got = _np(P.partial_mttkrp(xd, hs, "left", plan, sliced=sl).data)
    want = O.partial_left(x, dims, plan.split, hs)
    # mixed signs: the bound is relative to sum |x||b| (cancellation), checked per row
    absref = O.partial_left(np.abs(x), dims, plan.split, [np.abs(h) for h in hs])
    assert np.max(np.abs(got - want) / np.maximum(absref, 1e-300)) <= 1e-13
    got = _np(P.partial_mttkrp(xd, hs, "right", plan, sliced=sl).data)
    want = O.partial_right(x, dims, plan.split, hs)
    absref = O.partial_right(np.abs(x), dims, plan.split, [np.abs(h) for h in hs])
    assert np.max(np.abs(got - want) / np.maximum(absref, 1e-300)) <= 1e-13


def test_sliced_bitwise_reproducible(P):
    import torch

    from paper_1909_01149_b200 import synth

    dims, r = (640, 640, 320), 32
    fs = synth.truth_factors(dims, r, 3, "uniform")
    x = synth.synthetic_block(dims, fs, 0.01, 3)
    plan = P.DimTreePlan.create(dims, r)
    sl = _sliced(P, x, plan)
    hs = [torch.from_numpy(f).cuda() for f in fs]
    for side in ("left", "right"):
        a = P.partial_mttkrp(x, hs, side, plan, sliced=sl).data.clone()
        b = P.partial_mttkrp(x, hs, side, plan, sliced=sl).data.clone()
        assert torch.equal(a, b), side


def test_sliced_runs_vs_golden(P, golden):
    """Every golden sequential run (live reference traces) with the sliced engine forced."""
    g = golden("runs.npz")
    for name in [str(n) for n in g["names"]]:
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        algo = str(g[f"{name}_algo"])
        x = P.DenseTensor(dims, g[f"{name}_x"])
        cfg = P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed, mttkrp_kernel="sliced")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = P.nncp_sequential(x, cfg)
        ref = g[f"{name}_errors"]
        got = np.array(rep.errors)
        k = min(11, len(ref))
        assert np.max(np.abs(got[:k] - ref[:k])) <= TRACE_TOL, (name, np.max(np.abs(got[:k] - ref[:k])))
        for n in range(len(dims)):
            assert np.max(np.abs(rep.model.factors[n] - g[f"{name}_f{n}"])) <= FACTOR_TOL, (name, n)


@pytest.mark.parametrize("dims,r,algo,iters", [((128, 128, 128), 16, "hals", 8), ((32, 32, 32, 32), 32, "bpp", 4),
                                               ((256, 128, 16), 20, "hals", 6), ((96, 80, 64), 64, "mu", 5),
                                               ((128, 96, 80), 16, "nes", 10), ((64, 48, 40, 8), 8, "nes", 8),
                                               ((128, 96, 80), 16, "admm", 6)])
def test_sliced_runs_vs_oracle(P, dims, r, algo, iters):
    rng = np.random.default_rng(sum(dims) * r)
    hs = [rng.random((d, r)) for d in dims]
    x = O.reconstruct(hs, np.ones(r))
    x = x + 0.01 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))
    errors, factors, lam, _, _ = O.run_sequential(x, dims, r, algo, iters, 0.0, 0)
    rep = P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0,
                                                                mttkrp_kernel="sliced"))
    assert np.max(np.abs(np.array(rep.errors) - np.array(errors))) <= TRACE_TOL
    for a, b in zip(rep.model.factors, factors):
        assert np.max(np.abs(a - b)) <= FACTOR_TOL


def test_sliced_graph_matches_eager(P):
    rng = np.random.default_rng(11)
    dims, r = (160, 144, 120), 24
    hs = [rng.random((d, r)) for d in dims]
    x = O.reconstruct(hs, np.ones(r))
    runs = []
    for graph in (False, True):
        cfg = P.RunConfig(rank=r, algorithm="hals", max_iters=5, tol=0.0, cuda_graph=graph, mttkrp_kernel="sliced")
        runs.append(P.nncp_sequential(P.DenseTensor(dims, x), cfg))
    assert runs[0].errors == runs[1].errors
    for a, b in zip(runs[0].model.factors, runs[1].model.factors):
        assert np.array_equal(a, b)


def test_sliced_grid_runs_vs_golden(P, golden):
    """Thread-simulated grid runs (one engine, one sliced tensor block per worker) vs the reference's grid runs."""
    g = golden("runs.npz")
    for tag in [str(t) for t in g["grids"]]:
        name = tag[len("grid_"):tag.rindex("_")]
        grid = tuple(int(v) for v in tag[tag.rindex("_") + 1:].split("x"))
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        algo = str(g[f"{name}_algo"])
        x = P.DenseTensor(dims, g[f"{name}_x"])
        cfg = P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed, grid=grid,
                          mttkrp_kernel="sliced")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            par = P.nncp_parallel(x, cfg)
        assert np.max(np.abs(np.array(par.errors) - g[f"{tag}_errors"])) <= TRACE_TOL, tag
        for n in range(len(dims)):
            assert np.max(np.abs(par.model.factors[n] - g[f"{tag}_f{n}"])) <= FACTOR_TOL, (tag, n)


def test_sliced_seven_levels_run(P):
    """RunConfig.mttkrp_levels=7 (54-bit digit operands) through the whole driver."""
    rng = np.random.default_rng(21)
    dims, r = (96, 80, 64), 12
    hs = [rng.random((d, r)) for d in dims]
    x = O.reconstruct(hs, np.ones(r))
    errors, factors, _, _, _ = O.run_sequential(x, dims, r, "hals", 5, 0.0, 0)
    cfg = P.RunConfig(rank=r, algorithm="hals", max_iters=5, tol=0.0, mttkrp_kernel="sliced", mttkrp_levels=7)
    rep = P.nncp_sequential(P.DenseTensor(dims, x), cfg)
    assert np.max(np.abs(np.array(rep.errors) - np.array(errors))) <= TRACE_TOL
    for a, b in zip(rep.model.factors, factors):
        assert np.max(np.abs(a - b)) <= FACTOR_TOL
    with pytest.raises(ValueError, match="mttkrp_levels"):
        P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=r, mttkrp_levels=5))


@pytest.mark.parametrize("dims,r", [((1024, 300, 1024), 32), ((512, 600, 32, 32), 24), ((768, 400, 1030), 1)])
def test_fused_trailing_ttv(P, dims, r):
    """Left partial + first trailing TTV in one sliced pass == partial then multi_ttv (T_L bitwise, the
    mode-1 MTTKRP to 1e-12), and the mode-1 MTTKRP vs the oracle."""
    import torch

    from paper_1909_01149_b200.dimtree import fused_trailing_ok, partial_mttkrp_trailing

    rng = np.random.default_rng(sum(dims) * r)
    x = rng.random(int(np.prod(dims)))
    hs = [rng.random((d, r)) for d in dims]
    plan = P.DimTreePlan.create(dims, r)
    xd = P.DenseTensor(dims, x).to_device()
    sl = _sliced(P, xd, plan)
    assert fused_trailing_ok(plan, sl)
    ws = P.tensor_ops.Workspace(max(plan.workspace_bytes(), plan.sliced_workspace_bytes()))
    t_ref = P.partial_mttkrp(xd, hs, "left", plan, workspace=ws, sliced=sl).data.clone()
    m_ref = P.multi_ttv(P.dimtree.TempTensor(dims[:2], r, t_ref), hs[1:2], "trailing").data.clone()
    out_t = torch.empty_like(t_ref)
    out_m = torch.empty(dims[0] * r, dtype=torch.float64, device="cuda")
    partial_mttkrp_trailing(xd, hs, plan, sl, out_t, out_m, ws)
    assert torch.equal(out_t, t_ref)
    assert float(torch.linalg.norm(out_m - m_ref) / torch.linalg.norm(m_ref)) <= MTTKRP_TOL
    want = O.naive_mttkrp(x, dims, hs, 0)
    assert rel_fro(_np(out_m.view(r, dims[0]).T), want) <= MTTKRP_TOL


def test_sliced_balanced_split_run(P):
    """dimtree_split="auto": the sliced engine takes the split minimising M + J (4096 x 2048 x 256-like
    shapes: S = 1 instead of the reference's S = 2); same traces as the oracle and as the reference split."""
    rng = np.random.default_rng(31)
    dims, r = (192, 96, 24), 12
    hs = [rng.random((d, r)) for d in dims]
    x = O.reconstruct(hs, np.ones(r))
    errors, factors, _, _, _ = O.run_sequential(x, dims, r, "hals", 6, 0.0, 0)
    reps = {}
    for mode in ("auto", "reference"):
        cfg = P.RunConfig(rank=r, algorithm="hals", max_iters=6, tol=0.0, mttkrp_kernel="sliced", dimtree_split=mode)
        reps[mode] = P.nncp_sequential(P.DenseTensor(dims, x), cfg)
    assert reps["auto"].split_mode == 1 and reps["reference"].split_mode == 2
    for rep in reps.values():
        assert np.max(np.abs(np.array(rep.errors) - np.array(errors))) <= TRACE_TOL
        for a, b in zip(rep.model.factors, factors):
            assert np.max(np.abs(a - b)) <= FACTOR_TOL
    with pytest.raises(ValueError, match="dimtree_split"):
        P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=r, dimtree_split="middle"))


def test_sliced_balanced_split_grid_run(P):
    """Thread-simulated 2x2x1 grid on a skewed shape: every worker's block takes the balanced split
    (local 48x24x8: S = 1); the grid run matches the oracle's sequential run."""
    rng = np.random.default_rng(37)
    dims, r = (96, 48, 8), 6
    hs = [rng.random((d, r)) for d in dims]
    x = O.reconstruct(hs, np.ones(r))
    errors, factors, _, _, _ = O.run_sequential(x, dims, r, "hals", 6, 0.0, 0)
    cfg = P.RunConfig(rank=r, algorithm="hals", max_iters=6, tol=0.0, grid=(2, 2, 1), mttkrp_kernel="sliced")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        par = P.nncp_parallel(P.DenseTensor(dims, x), cfg)
    assert par.split_mode == 1
    assert np.max(np.abs(np.array(par.errors) - np.array(errors))) <= TRACE_TOL
    for a, b in zip(par.model.factors, factors):
        assert np.max(np.abs(a - b)) <= FACTOR_TOL


def _heavy_tailed(rng, dims, r, spikes=32):
    """Nonnegative rows with a few 2^20 spikes in slices where the contracted factor is zero:
    the outputs never see the spikes, but the row scale of the digit planes does."""
    x = rng.uniform(0.5, 1.0, int(np.prod(dims))).reshape(dims[2], -1)
    cols = rng.choice(dims[2], size=spikes, replace=False)
    x[cols, :] = 2.0 ** 20
    hs = [rng.random((d, r)) for d in dims]
    hs[2][cols, :] = 0.0
    return x.ravel(), hs


def _cancelling(rng, dims, r, k):
    """Signed rows x[m, j] = s_j (1 + 2^-k u): with factor rows equal in pairs and s_j
    alternating, the O(1) parts cancel exactly and the outputs are O(2^-k)."""
    m = int(np.prod(dims[:2]))
    s = np.where(np.arange(dims[2]) % 2 == 0, 1.0, -1.0)
    x = (s[:, None] * (1.0 + 2.0 ** -k * rng.random((dims[2], m)))).ravel()
    hs = [rng.random((d, r)) for d in dims]
    hs[2][1::2] = hs[2][0::2]
    return x, hs


def test_sliced_six_levels_failure_modes(P):
    """Where the 6-level Ozaki bound (relative to each row's maximum) does NOT give 1e-12
    on the outputs -- the cases "auto" routes to the fp64 engine: heavy-tailed rows whose
    spikes meet zero factor rows, and signed rows whose large parts cancel.  The fp64
    engine meets the tolerance on the same inputs."""
    dims, r = (64, 64, 4096), 16
    plan = P.DimTreePlan.create(dims, r)
    rng = np.random.default_rng(77)
    for name, (x, hs) in (("heavy-tailed", _heavy_tailed(rng, dims, r)),
                          ("cancelling", _cancelling(rng, dims, r, 10))):
        xd = P.DenseTensor(dims, x).to_device()
        want = O.partial_left(x, dims, plan.split, hs)
        fp64 = rel_fro(_np(P.partial_mttkrp(xd, hs, "left", plan).data), want)
        sl6 = rel_fro(_np(P.partial_mttkrp(xd, hs, "left", plan, sliced=_sliced(P, xd, plan, 6)).data), want)
        print(f"{name}: fp64 {fp64:.2e}  sliced-6 {sl6:.2e}")
        assert fp64 <= MTTKRP_TOL, (name, fp64)
        assert sl6 > MTTKRP_TOL, (name, sl6)   # the failure mode the engine choice guards against


@pytest.mark.parametrize("case", ["signed", "heavy-tailed", "ucp", "nonneg"])
def test_auto_engine_guards(P, case):
    """mttkrp_kernel="auto" at a size where the cost model picks the sliced engine:
    it slices only finite, nonnegative tensors of moderate dynamic range, and never for
    UCP's signed factors (driver._sliced_ok_for)."""
    from paper_1909_01149_b200.driver import _Engine
    from paper_1909_01149_b200.grid import IdentityCollectives

    dims, r = (512, 512, 256), 32                # 2^26 elements: sliced wins the cost model
    rng = np.random.default_rng(8)
    x = rng.uniform(0.5, 1.0, int(np.prod(dims)))
    algo = "hals"
    if case == "signed":
        x[::1000] = -1e-3
    elif case == "heavy-tailed":
        x[::100000] = 1e6
    elif case == "ucp":
        algo = "ucp"
    xd = P.DenseTensor(dims, x).to_device()
    eng = _Engine(xd.data, dims, dims, P.RunConfig(rank=r, algorithm=algo, max_iters=1), IdentityCollectives())
    sliced = eng.sliced is not None
    assert sliced == (case == "nonneg"), (case, eng.facts.min, eng.facts.dynamic_range)
    if case == "signed":
        assert eng.facts.signed
    del eng, xd


def test_non_finite_tensor_uses_fp64_engine(P):
    """NaN / Inf have no digits: even a forced sliced engine falls back (with a warning) and
    the NaN propagates into the error trace like the reference's arithmetic."""
    import torch

    from paper_1909_01149_b200.driver import _Engine
    from paper_1909_01149_b200.grid import IdentityCollectives

    dims, r = (40, 30, 20), 4
    x = np.random.default_rng(2).random(int(np.prod(dims)))
    x[123] = np.nan
    xd = torch.as_tensor(x, device="cuda")
    with pytest.warns(UserWarning, match="non-finite"):
        eng = _Engine(xd, dims, dims, P.RunConfig(rank=r, algorithm="hals", max_iters=1, mttkrp_kernel="sliced"),
                      IdentityCollectives())
    assert eng.sliced is None and not eng.facts.finite


@pytest.mark.parametrize("algo", ["hals", "mu", "bpp"])
@pytest.mark.parametrize("dims,side", [((256, 256, 128), "right"), ((300, 64, 48), "right"),
                                       ((1024, 256, 256), "left")])
def test_deferred_groups_feed_the_update_bitwise(P, algo, dims, side):
    """nncp_partial_mttkrp_sliced_deferred + nncp_update_grouped (the update sums the
    split-K group partials while loading its rows) == nncp_partial_mttkrp_sliced (group
    reduction kernel) + nncp_update_ex on the reduced temporary, bit for bit."""
    import torch

    from paper_1909_01149_b200 import _lib
    from paper_1909_01149_b200.dimtree import DeferredPartial
    from paper_1909_01149_b200.tensor_ops import Workspace

    r = 16
    rng = np.random.default_rng(sum(dims))
    x = P.DenseTensor(dims, rng.random(int(np.prod(dims)))).to_device()
    split = 1 if side == "left" else 2
    plan = P.DimTreePlan.create(dims, r) if split == 2 else P.DimTreePlan(dims=dims, rank=r, split=1)
    assert plan.split == split
    sl = _sliced(P, x, plan)
    hs = [torch.as_tensor(rng.random((d, r)), device="cuda") for d in dims]
    ws = Workspace(plan.sliced_workspace_bytes(6))
    mode = 0 if side == "left" else 2
    rows = dims[mode]
    d = P.partial_mttkrp(x, hs, side, plan, workspace=ws, sliced=sl, defer=True)
    assert isinstance(d, DeferredPartial) and d.groups > 1, "shape must split the contraction into groups"
    lib, st = _lib.load(), _lib.stream_handle()
    grams = torch.stack([h.T @ h for h in hs]).contiguous()
    cur = torch.as_tensor(rng.random((rows, r)), device="cuda")
    status = torch.zeros((2, _lib.STATUS_WORDS), dtype=torch.int32, device="cuda")
    uws = Workspace(1 << 22)
    outs = []
    for k in range(2):
        hhat = torch.empty((rows, r), dtype=torch.float64, device="cuda")
        nsq = torch.empty(r, dtype=torch.float64, device="cuda")
        beta = torch.zeros(1, dtype=torch.float64, device="cuda")
        sets = torch.zeros(rows, dtype=torch.int64, device="cuda") if algo == "bpp" else None
        if k == 0:
            _lib.check(lib.nncp_update_grouped(_lib.ALGO_CODES[algo], _lib.ptr(grams), 3, mode, r, d.ptr, rows,
                                               d.groups, d.gstride, _lib.ptr(cur), None, rows, _lib.ptr(hhat),
                                               _lib.ptr(nsq), _lib.ptr(beta), _lib.ptr(status[k]), 1e-16,
                                               _lib.ptr(sets) if sets is not None else None, uws.ptr, uws.nbytes,
                                               st))
        else:
            t = P.partial_mttkrp(x, hs, side, plan, workspace=ws, sliced=sl)
            _lib.check(lib.nncp_update_ex(_lib.ALGO_CODES[algo], _lib.ptr(grams), 3, mode, r, _lib.ptr(t.data),
                                          _lib.ptr(cur), None, rows, _lib.ptr(hhat), _lib.ptr(nsq), _lib.ptr(beta),
                                          _lib.ptr(status[k]), 1e-16,
                                          _lib.ptr(sets) if sets is not None else None, rows, uws.ptr, uws.nbytes,
                                          st))
        torch.cuda.synchronize()
        outs.append((hhat.cpu().numpy(), nsq.cpu().numpy(), beta.cpu().numpy()))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    # the group partials overlapping the update's own scratch are refused
    with pytest.raises(ValueError):
        _lib.check(lib.nncp_update_grouped(_lib.ALGO_CODES[algo], _lib.ptr(grams), 3, mode, r,
                                           _lib.vp(uws.ptr.value + 4096), rows, 2, rows * r, _lib.ptr(cur), None, rows,
                                           _lib.ptr(hhat), _lib.ptr(nsq), None, _lib.ptr(status[0]), 1e-16, None,
                                           uws.ptr, uws.nbytes, st))
