"""Edge of the device path's order range (NNCP_MAX_ORDER = 8): an 8-way tensor runs
HALS / MU / BPP on both MTTKRP engines and matches the oracle at the north-star
tolerances (traces <= 1e-9, factors <= 1e-6); order 9 is refused up front with a
clear error instead of reaching a kernel."""

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


@pytest.mark.parametrize("algo", ["hals", "mu", "bpp"])
@pytest.mark.parametrize("engine", ["fp64", "sliced"])
def test_eight_way_tensor_matches_oracle(P, algo, engine):
    dims, r = (4, 3, 3, 2, 3, 2, 5, 3), 5
    rng = np.random.default_rng(8)
    hs = [rng.random((d, r)) for d in dims]
    x = O.khatri_rao(hs) @ np.ones(r)
    x = x + 0.02 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))
    errors, factors, lam, _, _ = O.run_sequential(x, dims, r, algo, 6, 0.0, 0)
    rep = P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(rank=r, algorithm=algo, max_iters=6, tol=0.0,
                                                                mttkrp_kernel=engine))
    assert np.max(np.abs(np.array(rep.errors) - np.array(errors))) <= 1e-9
    for a, b in zip(rep.model.factors, factors):
        assert np.max(np.abs(a - b)) <= 1e-6
    # and the 8-way grid path (thread workers on the one GPU)
    par = P.nncp_parallel(P.DenseTensor(dims, x), P.RunConfig(rank=r, algorithm=algo, max_iters=6, tol=0.0,
                                                              grid=(2, 1, 1, 1, 1, 1, 1, 1), mttkrp_kernel=engine))
    assert np.max(np.abs(np.array(par.errors) - np.array(errors))) <= 1e-9


def test_order_nine_is_refused(P):
    dims = (2,) * 9
    with pytest.raises(NotImplementedError, match="order 9"):
        P.nncp_sequential(P.DenseTensor(dims, np.ones(2 ** 9)), P.RunConfig(rank=2, algorithm="mu", max_iters=1))
