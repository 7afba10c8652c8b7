"""ANLS-BPP on the device (bpp_kernel): each row's block principal
pivoting starts from the passive set it ended with in the previous outer iteration
(RunConfig.bpp_warm_start, default on), and a pass with few active variables solves
through S^-1 (Gauss-Jordan once per CTA) by block elimination instead of a
full LU of S[P,P].  The NNLS minimiser is unique for SPD S, so warm and cold starts
agree to rounding (bitwise when every pass is a direct solve), and both match the
reference's golden runs and the oracle; a row whose fast attempt fails is redone with
the reference's own cold-start direct solves."""

import warnings

import numpy as np
import pytest

from oracle import nncp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as pkg

    return pkg


def _run(P, x, dims, r, iters, seed, warm, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=r, algorithm="bpp", max_iters=iters,
                                                                    tol=0.0, seed=seed, bpp_warm_start=warm, **kw))


def test_warm_start_matches_cold_start_on_golden_runs(P, golden):
    g = golden("runs.npz")
    names = [n for n in (str(v) for v in g["names"]) if str(g[f"{n}_algo"]) == "bpp"]
    assert names
    for name in names:
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        warm = _run(P, g[f"{name}_x"], dims, r, iters, iseed, True)
        cold = _run(P, g[f"{name}_x"], dims, r, iters, iseed, False)
        assert np.max(np.abs(np.array(warm.errors) - np.array(cold.errors))) <= 1e-13, name
        for a, b in zip(warm.model.factors, cold.model.factors):
            assert np.max(np.abs(a - b)) <= 1e-12, name
        assert np.max(np.abs(np.array(warm.errors) - g[f"{name}_errors"])) <= 1e-9, name


@pytest.mark.parametrize("dims,r,iters", [((64, 48, 40, 24), 16, 12), ((128, 128, 64), 32, 10), ((90, 80, 70), 64, 6)])
def test_warm_start_matches_cold_start_and_oracle(P, dims, r, iters):
    rng = np.random.default_rng(sum(dims) + r)
    hs = [rng.random((d, r)) for d in dims]
    x = O.khatri_rao(hs) @ np.ones(r)
    x += 0.01 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))
    warm = _run(P, x, dims, r, iters, 0, True)
    cold = _run(P, x, dims, r, iters, 0, False)
    same = all(np.array_equal(a, b) for a, b in zip(warm.model.factors, cold.model.factors))
    print(f"{dims} R={r}: warm == cold bitwise: {same}")
    assert np.max(np.abs(np.array(warm.errors) - np.array(cold.errors))) <= 1e-13
    errors, factors, _, _, _ = O.run_sequential(x, dims, r, "bpp", iters, 0.0, 0, init_error="tree")
    assert np.max(np.abs(np.array(warm.errors[:11]) - np.array(errors[:11]))) <= 1e-9
    for a, b in zip(warm.model.factors, factors):
        assert np.max(np.abs(a - b)) <= 1e-6


def test_warm_start_in_graph_replays_and_grid(P, golden):
    """The passive sets live in device buffers captured by the sweep graph; the thread
    grid keeps one set per owned row on every worker."""
    g = golden("runs.npz")
    name = "bpp3"
    dims = tuple(int(d) for d in g[f"{name}_dims"])
    r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
    eager = _run(P, g[f"{name}_x"], dims, r, iters, iseed, True, cuda_graph=False)
    graph = _run(P, g[f"{name}_x"], dims, r, iters, iseed, True)
    assert eager.errors == graph.errors
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        par = P.nncp_parallel(P.DenseTensor(dims, g[f"{name}_x"]),
                              P.RunConfig(rank=r, algorithm="bpp", max_iters=iters, tol=0.0, seed=iseed, grid=(2, 2, 1)))
    assert np.max(np.abs(np.array(par.errors) - np.array(eager.errors))) <= 1e-12
