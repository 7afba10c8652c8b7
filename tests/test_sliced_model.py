"""The sliced-tensor MTTKRP algorithm (tests/sliced_model.py, a bit-exact model of
the int8 tensor-core kernels) against the oracle on the CPU, and the CUDA
kernels against the model bit for bit on the GPU."""

import numpy as np
import pytest

from oracle import nncp_oracle as O
from tests.conftest import rel_fro
from tests.sliced_model import plan, sliced_partial

MTTKRP_TOL = 1e-12

CASES = [((7, 9, 11), 5), ((33, 17, 5), 1), ((96, 64, 48), 20), ((256, 130, 40), 8), ((128, 24, 30, 8), 12),
         ((20, 18, 16, 14), 33), ((256, 256, 64), 8), ((40, 40, 20000), 4),
         ((128, 16, 16, 200), 4),   # split 3: right side = 3 Khatri-Rao factors, segment-reuse path
         ((300, 260, 90), 64), ((256, 128, 96), 50),   # RP = 64
         # balanced root split S = 1 (driver: dimtree_split="auto"): the left side has a few
         # row tiles over a long contraction -> split-K groups on the left
         ((64, 96, 300), 20, 1), ((256, 128, 64), 12, 1), ((40, 300, 200), 33, 1)]


def _split(case):
    from paper_1909_01149_b200.dimtree import choose_split_mode

    return case[2] if len(case) > 2 else choose_split_mode(case[0])


def _case(dims, r, signed=False):
    rng = np.random.default_rng(sum(dims) * 7 + r)
    x = rng.random(int(np.prod(dims)))
    hs = [rng.random((d, r)) for d in dims]
    if signed:
        x = x - 0.4
        hs = [h - 0.3 for h in hs]
    return x, hs


# the CPU model runs exact int64 matmuls in numpy: keep the CPU suite to the smaller cases
CPU_CASES = [c for c in CASES if np.prod(c[0]) * c[1] <= 3e7]


@pytest.mark.parametrize("case", CPU_CASES, ids=str)
def test_model_matches_oracle(case):
    dims, r = case[:2]
    x, hs = _case(dims, r)
    s = _split(case)
    for side, fn in (("left", O.partial_left), ("right", O.partial_right)):
        got = sliced_partial(x, dims, s, side, hs, r)
        assert rel_fro(got, fn(x, dims, s, hs)) <= MTTKRP_TOL, (side, dims, r)


def test_model_levels7_and_signs():
    dims, r = (96, 64, 48), 20
    x, hs = _case(dims, r, signed=True)
    for levels, tol in ((6, 1e-12), (7, 1e-14)):
        for side, fn in (("left", O.partial_left), ("right", O.partial_right)):
            got = sliced_partial(x, dims, 2, side, hs, r, levels=levels)
            want = fn(x, dims, 2, hs)
            absref = fn(np.abs(x), dims, 2, [np.abs(h) for h in hs])
            assert np.max(np.abs(got - want) / absref) <= tol, (levels, side)


def test_plan_splits_contraction_evenly():
    p = plan((2048, 2048, 2048), 2, "right", 32)
    assert p["groups"] == 9 and p["nchunks"] % p["groups"] == 0 and p["Kc"] <= 16384
    p = plan((1024, 1024, 1024), 2, "right", 32)
    assert p["groups"] == 18 and p["nchunks"] % p["groups"] == 0
    p = plan((2048, 2048, 2048), 2, "left", 32)
    assert p["groups"] == 1 and p["nchunks"] == 1
    p = plan((40, 40, 20000), 2, "left", 4)          # 13 row tiles: split-K groups on the left too
    assert p["groups"] == 10 and p["nchunks"] == 10
    p = plan((4096, 2048, 256), 1, "left", 20)       # c4 under the balanced split
    assert p["groups"] == 4 and p["nchunks"] % p["groups"] == 0


def test_balanced_split():
    from paper_1909_01149_b200.dimtree import choose_balanced_split
    from paper_1909_01149_b200.driver import _split_rows

    assert choose_balanced_split((4096, 2048, 256)) == 1
    assert choose_balanced_split((256, 256, 256, 256)) == 2
    assert choose_balanced_split((40, 40, 20000)) == 2
    assert choose_balanced_split((30, 20)) == 1
    # the engine switches only when M + J at least halves: never for cubes
    assert 2 * _split_rows((4096, 2048, 256), 1) <= _split_rows((4096, 2048, 256), 2)
    assert 2 * _split_rows((512, 512, 512), 1) > _split_rows((512, 512, 512), 2)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=str)
def test_kernels_bitwise_equal_model(case):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200 import _lib
    from paper_1909_01149_b200.dimtree import SlicedTensor

    dims, r = case[:2]
    sms = _lib.load().nncp_device_sms()
    x, hs = _case(dims, r, signed=(r % 2 == 1))
    plan_ = P.DimTreePlan(tuple(dims), r, _split(case))
    xd = P.DenseTensor(dims, x).to_device()
    sl = SlicedTensor(xd, dims, plan_.split)
    for side in ("left", "right"):
        got = P.partial_mttkrp(xd, hs, side, plan_, sliced=sl).data.cpu().numpy()
        want = sliced_partial(x, dims, plan_.split, side, hs, r, sms=sms)
        assert np.array_equal(got, want), (side, dims, r, float(np.max(np.abs(got - want))))
