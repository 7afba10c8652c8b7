"""The C-ABI library loads on a CPU-only host and exports every declared symbol."""

import ctypes
import os
import re

from tests.conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "nncp_b200.h")).read()
    return sorted(set(re.findall(r"\b(nncp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1909_01149_b200 import _lib

    lib = _lib.load(require_device=False)
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert bound == set(names)


def test_pure_host_entry_points():
    from paper_1909_01149_b200 import _lib

    lib = _lib.load(require_device=False)
    assert lib.nncp_abi_version() == 1
    out = ctypes.c_int(0)
    assert lib.nncp_choose_split(3, _lib.i64([128, 128, 128]), 0, ctypes.byref(out)) == 0 and out.value == 2
    assert lib.nncp_choose_split(4, _lib.i64([384] * 4), 1, ctypes.byref(out)) == 0 and out.value == 3
    assert lib.nncp_choose_split(3, _lib.i64([1446680, 69, 25]), 0, ctypes.byref(out)) == 0 and out.value == 1
    assert lib.nncp_choose_split(3, _lib.i64([2, 2, 100]), 0, ctypes.byref(out)) == 0 and out.value == 2
    assert lib.nncp_workspace_bytes(3, _lib.i64([2048] * 3), 2, 32) > 0
    # BPP passive sets + the prepared S / S^-1 block: rows rounded up to 2, 4 header words, 2 R^2
    assert lib.nncp_bpp_sets_words(255, 32) == 256 + 4 + 2 * 32 * 32
    assert lib.nncp_bpp_sets_words(0, 5) == 4 + 2 * 25
    assert lib.nncp_bpp_prepare(None, 3, 3, 8, None, 10, None) != 0          # mode out of range
    assert lib.nncp_bpp_prepare(None, 3, 0, 8, None, -1, None) != 0          # negative rows


def test_device_calls_fail_loudly_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1909_01149_b200 as P

    with pytest.raises(RuntimeError, match="CUDA device"):
        P.gram([[1.0, 2.0], [3.0, 4.0]])


def test_sliced_sizing_entry_points():
    """Host-side sizing / validation of the sliced (int8 tensor-core) MTTKRP path."""
    from paper_1909_01149_b200 import _lib
    from paper_1909_01149_b200.dimtree import DimTreePlan, SlicedTensor

    lib = _lib.load(require_device=False)
    # 2048^3, split 2: int32 row exponents + uint64 row maxima + 6 planes of 128x128-blocked digits
    m, j = 2048 * 2048, 2048
    expect = 1024 + (m * 4 + m * 8) + 6 * m * j
    assert SlicedTensor.nbytes((2048, 2048, 2048), 2) == expect
    assert SlicedTensor.nbytes((2048, 2048, 2048), 2, levels=7) == expect + m * j
    # padding of ragged unfoldings to whole 128 x 128 blocks
    assert SlicedTensor.nbytes((7, 9, 11), 2) >= 6 * 128 * 128
    p = DimTreePlan.create((2048, 2048, 2048), 32)
    ws = p.sliced_workspace_bytes()
    # right side: factor digits 6 x 32 x M bytes dominate
    assert 6 * 32 * m <= ws < 6 * 32 * m + (64 << 20)
    assert lib.nncp_sliced_workspace_bytes(3, _lib.i64([64, 64, 64]), 0, 8, 6) == 0     # bad split
    out = ctypes.c_size_t(0)
    assert lib.nncp_sliced_tensor_bytes(3, _lib.i64([64, 64, 64]), 2, 5, ctypes.byref(out)) == _lib.NNCP_ERR_UNSUPPORTED
    assert lib.nncp_sliced_tensor_bytes(3, _lib.i64([64, 64, 64]), 3, 6, ctypes.byref(out)) == _lib.NNCP_ERR_VALUE
