"""The reference's acceptance criteria (SPEC §ACCEPTANCE, pkg/tests/test_acceptance.py) re-run on the device."""

import time
import warnings

import numpy as np
import pytest

from oracle import nncp_oracle as O

pytestmark = pytest.mark.gpu


def _host(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as pkg

    return pkg


def test_c01_dimension_tree_oracle_equivalence(P):
    """test_acceptance.py:48-66: 200 random instances, every mode, max-abs within 1e-12 of the naive MTTKRP."""
    rng = np.random.default_rng(101)
    t0 = time.perf_counter()
    for _ in range(200):
        order = int(rng.integers(3, 6))
        dims = tuple(int(d) for d in rng.integers(2, 7, size=order))
        rank = int(rng.integers(1, 5))
        x = rng.standard_normal(int(np.prod(dims)))
        hs = [rng.standard_normal((d, rank)) for d in dims]
        ctx = P.DimTreeContext(P.DimTreePlan.create(dims, rank))
        ctx.begin_iteration()
        xd = P.DenseTensor(dims, x).to_device()
        for mode in range(order):
            got = _host(ctx.mttkrp(xd, hs, mode))
            want = O.naive_mttkrp(x, dims, hs, mode)
            scale = max(np.abs(want).max(), 1e-30)
            assert np.abs(got - want).max() <= 1e-12 * scale
    assert time.perf_counter() - t0 < 60.0


def test_c02_two_partials_per_outer_iteration(P):
    rng = np.random.default_rng(102)
    for order in (2, 3, 4, 5, 6):
        dims = (3,) * order
        xd = P.DenseTensor(dims, rng.random(3 ** order)).to_device()
        hs = [rng.random((3, 2)) for _ in range(order)]
        ctx = P.DimTreeContext(P.DimTreePlan.create(dims, 2))
        for sweep in range(1, 4):
            ctx.begin_iteration()
            for mode in range(order):
                ctx.mttkrp(xd, hs, mode)
            assert ctx.partial_calls == 2 * sweep


def test_c05_bpp_matches_enumeration(P):
    """test_acceptance.py:150-187 (R <= 8, 100 instances)."""
    rng = np.random.default_rng(105)
    from tests.test_gpu_parity import _np

    for _ in range(100):
        r = int(rng.integers(1, 9))
        a = rng.standard_normal((r + 4, r))
        s = a.T @ a
        f = rng.standard_normal(r) * 2.0
        got = _np(P.bpp_update(P.UpdateInputs(s, f[None, :], np.zeros((1, r)))))[0]
        want = O.bpp_row(s, f, 0)
        assert np.allclose(got, want, atol=1e-8)
        y = s @ got - f
        scale = max(1.0, np.abs(f).max())
        assert (got >= 0).all()
        assert (y >= -1e-10 * scale).all()
        assert (np.abs(got * y) <= 1e-10 * scale * scale).all()


def test_c06_mu_objective_monotone(P):
    rng = np.random.default_rng(106)
    for _ in range(100):
        r = int(rng.integers(1, 6))
        a = rng.random((r + 4, r))
        b = rng.random((r + 4, 4))
        s, m = a.T @ a, b.T @ a
        h0 = rng.random((4, r)) + 1e-3
        h1 = _host(P.mu_update(P.UpdateInputs(s, m, h0)))
        f0 = np.linalg.norm(a @ h0.T - b) ** 2
        f1 = np.linalg.norm(a @ h1.T - b) ** 2
        assert f1 <= f0 * (1 + 1e-12) + 1e-12


def test_c07_error_identity_matches_reconstruction(P):
    rng = np.random.default_rng(107)
    for _ in range(100):
        order = int(rng.integers(2, 5))
        dims = tuple(int(d) for d in rng.integers(2, 9, size=order))
        while int(np.prod(dims)) > 4096:
            dims = dims[:-1] if len(dims) > 2 else (4, 4)
        rank = int(rng.integers(1, 4))
        x = rng.random(int(np.prod(dims))) + 0.01
        hs, lam = [], rng.random(rank) + 0.1
        for d in dims:
            h, w = O.normalize_columns(rng.random((d, rank)) + 0.05)
            lam = lam * w
            hs.append(h)
        last = len(dims) - 1
        ctx = P.DimTreeContext(P.DimTreePlan.create(dims, rank))
        m_n = _host(ctx.mttkrp_last_mode(P.DenseTensor(dims, x), hs))
        grams = [O.gram(h) for h in hs]
        s_n = O.hadamard_excluding(grams, last)
        eps = P.relative_error(float(x @ x), m_n, hs[last] * lam, s_n, grams[last], lam)
        assert abs(eps - O.relative_error_direct(x, hs, lam)) <= 1e-8


def test_c03_sequential_parallel_equivalence(P):
    """test_acceptance.py:88-107: 6 algorithms x 4 grids within 1e-10."""
    x, _ = P.generate_synthetic(P.SyntheticSpec((8, 8, 8), 2, seed=7))
    for algo in ("ucp", "mu", "hals", "bpp", "admm", "nes"):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            seq = P.nncp_sequential(x, P.RunConfig(rank=2, algorithm=algo, max_iters=8, tol=0.0, seed=5))
            for grid in [(1, 1, 1), (2, 1, 1), (2, 2, 2), (1, 4, 2)]:
                par = P.nncp_parallel(x, P.RunConfig(rank=2, algorithm=algo, max_iters=8, tol=0.0, seed=5,
                                                     grid=grid))
                assert len(par.errors) == len(seq.errors)
                diff = np.abs(np.array(par.errors) - np.array(seq.errors)).max()
                assert diff <= 1e-10, (algo, grid, diff)


def test_c08_communication_accounting(P):
    """test_acceptance.py:232-267: per-iteration collective volumes match the cost model exactly."""
    dims, rank, p = (8, 8, 8), 2, 8
    x, _ = P.generate_synthetic(P.SyntheticSpec(dims, rank, seed=108))

    def counters_for(iters, grid):
        return P.nncp_parallel(x, P.RunConfig(rank=rank, algorithm="bpp", max_iters=iters, tol=0.0, seed=1,
                                              grid=grid)).counters

    for grid in [(2, 2, 2), (2, 4, 1)]:
        one, two = counters_for(1, grid), counters_for(2, grid)

        def delta(field, name):
            return getattr(two, field).get(name, 0) - getattr(one, field).get(name, 0)

        per_mode = sum(rank * dims[n] // grid[n] for n in range(3))
        assert delta("words_in", "ReduceScatter") // p == per_mode
        assert delta("words_out", "AllGather") // p == per_mode
        assert delta("words_in", "AllReduce") // p == 3 * (rank ** 2 + rank) + 1
        assert delta("calls", "ReduceScatter") == 3 * p and delta("calls", "AllGather") == 3 * p
        assert delta("calls", "AllReduce") == (3 * 2 + 1) * p


def test_c09_collective_determinism(P):
    x, _ = P.generate_synthetic(P.SyntheticSpec((8, 8, 8), 2, seed=3))
    cfg = P.RunConfig(rank=2, algorithm="hals", max_iters=10, tol=0.0, seed=3, grid=(2, 2, 1))
    a, b = P.nncp_parallel(x, cfg), P.nncp_parallel(x, cfg)
    for fa, fb in zip(a.model.factors, b.model.factors):
        assert fa.tobytes() == fb.tobytes()
    assert a.model.lam.tobytes() == b.model.lam.tobytes()
