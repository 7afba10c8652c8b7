"""nncp_norm_rowmax + nncp_slice_tensor_planes (the init-row facts and the slicing row
maxima in one read of X): the sliced buffer is bitwise the one
nncp_slice_tensor writes, min x / max |x| / min nonzero |x| equal nncp_norm_squared_min's
exactly, and sum x^2 agrees to rounding (another summation order)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1909_01149_b200 import _lib

    return torch, _lib, _lib.load()


CASES = [((300, 70, 50), 2, "pos"), ((128, 96, 80), 1, "signed"), ((33, 17, 5, 7), 2, "pos"),
         ((257, 129, 65), 2, "wide"), ((512, 512, 64), 2, "pos"), ((64, 48, 40, 24), 3, "zeros"),
         ((40, 40, 20000), 2, "pos"), ((20, 30, 10), 1, "nan")]


@pytest.mark.parametrize("dims,split,kind", CASES)
@pytest.mark.parametrize("levels", [6, 7])
def test_norm_rowmax_then_planes_equals_slicing_at_once(env, dims, split, kind, levels):
    torch, _lib, lib = env
    rng = np.random.default_rng(sum(dims) + split)
    n = int(np.prod(dims))
    x = rng.random(n)
    if kind == "signed":
        x -= 0.5
    elif kind == "wide":
        x *= np.exp2(rng.integers(-30, 30, size=n))
    elif kind == "zeros":
        x[rng.random(n) < 0.3] = 0.0
    elif kind == "nan":
        x[n // 3] = np.nan
    xd = torch.as_tensor(x, device="cuda")
    nb = _lib.ctypes.c_size_t(0)
    _lib.check(lib.nncp_sliced_tensor_bytes(len(dims), _lib.i64(dims), split, levels, _lib.ctypes.byref(nb)))
    a = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    b = torch.full((nb.value,), 0x5A, dtype=torch.uint8, device="cuda")     # stale bytes must not matter
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    st = _lib.stream_handle()
    _lib.check(lib.nncp_slice_tensor(_lib.ptr(xd), len(dims), _lib.i64(dims), split, levels, _lib.ptr(a), nb.value, st))
    s_new = torch.zeros(4, dtype=torch.float64, device="cuda")
    s_old = torch.zeros(4, dtype=torch.float64, device="cuda")
    _lib.check(lib.nncp_norm_rowmax(_lib.ptr(xd), len(dims), _lib.i64(dims), split, levels, _lib.ptr(b), nb.value,
                                    _lib.ptr(s_new), _lib.vp(s_new.data_ptr() + 8), _lib.vp(ws.data_ptr()), ws.numel(),
                                    st))
    _lib.check(lib.nncp_slice_tensor_planes(_lib.ptr(xd), len(dims), _lib.i64(dims), split, levels, _lib.ptr(b),
                                            nb.value, st))
    _lib.check(lib.nncp_norm_squared_min(_lib.ptr(xd), n, _lib.ptr(s_old), _lib.vp(s_old.data_ptr() + 8),
                                         _lib.vp(ws.data_ptr()), ws.numel(), st))
    torch.cuda.synchronize()
    # the written regions, from each buffer's first 1 KB boundary: row exponents, row
    # maxima, digit planes (alignment gaps in between are never written)
    m = int(np.prod(dims[:split]))
    j = int(np.prod(dims[split:]))
    mp, jp = -(-m // 128) * 128, -(-j // 128) * 128
    rmax_off = -(-mp * 4 // 1024) * 1024
    plane_off = rmax_off + -(-mp * 8 // 1024) * 1024
    for buf in (a, b):
        assert buf.data_ptr() % 256 == 0
    oa, ob = (-a.data_ptr()) % 1024, (-b.data_ptr()) % 1024
    for lo, hi in ((0, mp * 4), (rmax_off, rmax_off + mp * 8), (plane_off, plane_off + levels * mp * jp)):
        assert torch.equal(a[oa + lo:oa + hi], b[ob + lo:ob + hi]), (lo, hi)
    new, old = s_new.cpu().numpy(), s_old.cpu().numpy()
    if kind == "nan":
        assert np.isnan(new[2]) and np.isnan(old[2])
        assert np.isnan(new[0]) and np.isnan(old[0])
        return
    assert np.array_equal(new[1:], old[1:])
    assert abs(new[0] - old[0]) <= 1e-14 * old[0]
    assert abs(new[0] - np.sum(x * x)) <= 1e-13 * new[0]
