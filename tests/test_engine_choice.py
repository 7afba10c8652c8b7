"""Host logic of the "auto" MTTKRP engine choice (no GPU): which tensors the sliced
int8 engine may take (driver._sliced_ok_for, DESIGN.md §4.4 "Engine choice")."""

import math

import pytest

from paper_1909_01149_b200.driver import SLICED_MAX_RANGE, TensorFacts, _sliced_ok_for, _use_sliced


def facts(alpha=1.0, xmin=0.0, absmax=1.0, absmin_nz=0.5):
    return TensorFacts(alpha, xmin, absmax, absmin_nz)


def test_nonnegative_moderate_range_may_slice():
    assert _sliced_ok_for(facts(), "hals") is None
    assert _sliced_ok_for(facts(absmax=SLICED_MAX_RANGE, absmin_nz=1.0), "bpp") is None
    assert _sliced_ok_for(facts(absmax=0.0, absmin_nz=math.inf), "mu") is None     # zero tensor: no range


@pytest.mark.parametrize("f,algo,why", [
    (facts(xmin=-1e-300), "hals", "negative"),
    (facts(), "ucp", "signed"),
    (facts(absmax=1.0, absmin_nz=0.5 / SLICED_MAX_RANGE), "hals", "span"),
    (facts(alpha=math.inf), "hals", "non-finite"),
    (facts(absmax=math.nan), "mu", "non-finite"),
])
def test_guarded_tensors_stay_on_fp64(f, algo, why):
    assert why in _sliced_ok_for(f, algo)
    # "auto" never slices them, whatever the size; an explicit "fp64" never slices
    assert not _use_sliced("auto", (4096, 4096, 4096), 2, 32, None, facts=f, algorithm=algo)
    assert not _use_sliced("fp64", (4096, 4096, 4096), 2, 32, None, facts=f, algorithm=algo)


def test_explicit_sliced_honoured_unless_non_finite():
    assert _use_sliced("sliced", (8, 8, 8), 2, 4, None, facts=facts(xmin=-1.0), algorithm="hals")
    with pytest.warns(UserWarning, match="non-finite"):
        assert not _use_sliced("sliced", (8, 8, 8), 2, 4, None, facts=facts(alpha=math.nan), algorithm="hals")


def test_small_tensors_stay_on_fp64():
    assert not _use_sliced("auto", (64, 64, 64), 2, 10, None, facts=facts(), algorithm="mu")
