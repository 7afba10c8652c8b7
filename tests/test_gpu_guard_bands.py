"""Out-of-bounds write checks for the hot kernels (compute-sanitizer is closed on this
GPU pool: runs under it left GPUs needing a reset -- profiles/r02_compute_sanitizer_closed.txt).

Every output a kernel writes -- MTTKRP temporaries (both engines, both sides, odd and
multi-chunk shapes), TTV results, update rows, column sums, beta, normalised rows, the
Grams, the end-of-sweep status codes, Khatri-Rao rows -- is placed inside a larger
buffer whose guard bands hold a NaN canary; the workspace gets a byte canary past the
size the call is told.  After the launch the results must match the oracle AND every
canary must be intact: a write one element past any edge, or past the workspace the
caller granted, fails the test.  Run-to-run bitwise reproducibility (the race check
the stress tests already apply to the mbarrier/TMA pipelines) is asserted as well."""

import numpy as np
import pytest

from oracle import nncp_oracle as O
from tests.conftest import rel_fro

pytestmark = pytest.mark.gpu

PAD = 64          # doubles of guard on each side (keeps the 512-byte allocation alignment)


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200 import _lib

    return P, _lib, torch


class Guarded:
    """A float64 device view with NaN guard bands on both sides."""

    def __init__(self, torch, n, fill=0.0):
        self.buf = torch.full((n + 2 * PAD,), float("nan"), dtype=torch.float64, device="cuda")
        self.view = self.buf[PAD:PAD + n]
        self.view.fill_(fill)
        self.n = n

    def intact(self):
        import torch

        torch.cuda.synchronize()
        head, tail = self.buf[:PAD], self.buf[PAD + self.n:]
        return bool(torch.isnan(head).all().item() and torch.isnan(tail).all().item())


class GuardedWs:
    """A workspace whose bytes past ``nbytes`` hold a 0x7F canary."""

    def __init__(self, torch, nbytes):
        self.nbytes = int(nbytes)
        self.buf = torch.zeros(self.nbytes + 4096, dtype=torch.uint8, device="cuda")
        self.buf[self.nbytes:] = 0x7F
        self.ptr = self.buf.data_ptr()

    def intact(self):
        import torch

        torch.cuda.synchronize()
        return bool((self.buf[self.nbytes:] == 0x7F).all().item())


@pytest.mark.parametrize("engine", ["fp64", "sliced"])
@pytest.mark.parametrize("dims,r", [((7, 9, 11), 5), ((33, 17, 5), 1), ((64, 32, 16500), 32),
                                    ((257, 129, 65), 33), ((30, 20, 10, 8), 12), ((100, 64, 64), 64)])
def test_partial_mttkrp_guard_bands(env, engine, dims, r):
    P, _lib, torch = env
    from paper_1909_01149_b200.dimtree import SlicedTensor

    rng = np.random.default_rng(sum(dims) + r)
    x = rng.random(int(np.prod(dims)))
    hs = [rng.random((d, r)) for d in dims]
    plan = P.DimTreePlan.create(dims, r)
    xd = P.DenseTensor(dims, x).to_device()
    sl = SlicedTensor(xd, dims, plan.split, 6) if engine == "sliced" else None
    need = plan.sliced_workspace_bytes(6) if sl is not None else plan.workspace_bytes()
    lib = _lib.load()
    s = plan.split
    dev = [torch.as_tensor(h, device="cuda") for h in hs]
    for side, fn, code in (("left", O.partial_left, _lib.SIDE_LEFT), ("right", O.partial_right, _lib.SIDE_RIGHT)):
        n = int(np.prod(dims[:s] if side == "left" else dims[s:])) * r
        outs = []
        for rep in range(2):
            out = Guarded(torch, n, fill=float(rep + 1))
            ws = GuardedWs(torch, need)
            used = range(s, len(dims)) if side == "left" else range(0, s)
            fac = _lib.ptrs([dev[m] if m in used else None for m in range(len(dims))])
            if sl is not None:
                _lib.check(lib.nncp_partial_mttkrp_sliced(_lib.ptr(sl.buf), len(dims), _lib.i64(dims), s, code, fac,
                                                          r, 6, _lib.ptr(out.view), _lib.vp(ws.ptr), ws.nbytes,
                                                          _lib.stream_handle()))
            else:
                _lib.check(lib.nncp_partial_mttkrp(_lib.ptr(xd.data), len(dims), _lib.i64(dims), s, code, fac, r,
                                                   _lib.ptr(out.view), _lib.vp(ws.ptr), ws.nbytes,
                                                   _lib.stream_handle()))
            assert out.intact(), (engine, dims, r, side, "output guard band overwritten")
            assert ws.intact(), (engine, dims, r, side, "write past the granted workspace")
            outs.append(out.view.cpu().numpy())
        assert rel_fro(outs[0], fn(x, dims, s, hs)) <= 1e-12, (engine, side)
        assert np.array_equal(outs[0], outs[1]), (engine, side, "not bitwise reproducible")


@pytest.mark.parametrize("side", ["trailing", "leading"])
@pytest.mark.parametrize("lead,rest,r", [(7, 5, 3), (129, 65, 8), (2, 4097, 1), (1025, 3, 33)])
def test_multi_ttv_guard_bands(env, side, lead, rest, r):
    P, _lib, torch = env
    rng = np.random.default_rng(lead + rest)
    t = rng.random(lead * rest * r)
    coeff = rng.random((rest if side == "trailing" else lead, r))
    n = (lead if side == "trailing" else rest) * r
    out = Guarded(torch, n)
    temp = P.TempTensor((lead, rest), r, torch.as_tensor(t, device="cuda"))
    P.multi_ttv(temp, torch.as_tensor(coeff, device="cuda"), side, out=out.view)
    assert out.intact()
    want = O.ttv_trailing(t, lead, r, coeff) if side == "trailing" else O.ttv_leading(t, lead, r, coeff)
    assert rel_fro(out.view.cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("algo", ["mu", "hals", "bpp", "ucp"])
@pytest.mark.parametrize("rows,r", [(1, 1), (37, 5), (1000, 32), (333, 64)])
def test_update_normalize_gram_guard_bands(env, algo, rows, r):
    P, _lib, torch = env
    lib = _lib.load()
    rng = np.random.default_rng(rows * r)
    order = 3
    grams = [rng.random((r + 3, r)) for _ in range(order)]
    g = np.stack([a.T @ a for a in grams])
    m = np.abs(rng.standard_normal((rows, r)))
    cur = rng.random((rows, r))
    st = _lib.stream_handle()
    dg = torch.as_tensor(g, device="cuda")
    dm = torch.as_tensor(m, device="cuda")
    dc = torch.as_tensor(cur, device="cuda")
    hhat, nsq, beta = Guarded(torch, rows * r), Guarded(torch, r), Guarded(torch, 1)
    status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device="cuda")
    _lib.check(lib.nncp_status_reset(_lib.ptr(status), st))
    ws = GuardedWs(torch, int(lib.nncp_workspace_bytes(order, _lib.i64((rows, 1, 1)), 1, r)))
    _lib.check(lib.nncp_update(_lib.ALGO_CODES[algo], _lib.ptr(dg), order, order - 1, r, _lib.ptr(dm), _lib.ptr(dc),
                               None, rows, _lib.ptr(hhat.view), _lib.ptr(nsq.view), _lib.ptr(beta.view),
                               _lib.ptr(status), _lib.vp(ws.ptr), ws.nbytes, st))
    assert hhat.intact() and nsq.intact() and beta.intact() and ws.intact(), algo
    s = g[0] * g[1]
    want = {"mu": O.mu_update, "hals": O.hals_update, "bpp": O.bpp_update, "ucp": O.ucp_update}[algo](s, m, cur)
    h = hhat.view.cpu().numpy().reshape(rows, r)
    assert rel_fro(h, want) <= 1e-10, algo
    assert rel_fro(nsq.view.cpu().numpy(), np.sum(want * want, axis=0)) <= 1e-10
    # normalise + Gram of the normalised rows, with guard bands on every output
    owned, lam, gout = Guarded(torch, rows * r), Guarded(torch, r), Guarded(torch, r * r)
    _lib.check(lib.nncp_normalize_gram(_lib.ptr(hhat.view), _lib.ptr(nsq.view), rows, r, _lib.ptr(owned.view),
                                       _lib.ptr(lam.view), _lib.ptr(gout.view), _lib.vp(ws.ptr), ws.nbytes, st))
    assert owned.intact() and lam.intact() and gout.intact() and ws.intact()
    hn, w = O.normalize_columns(h)
    assert rel_fro(owned.view.cpu().numpy().reshape(rows, r), hn) <= 1e-12
    assert rel_fro(gout.view.cpu().numpy().reshape(r, r), hn.T @ hn) <= 1e-12
    # the grid path's normalisation from an All-Reduced raw Gram
    graw = torch.as_tensor(h.T @ h, device="cuda")
    owned2, lam2, g2 = Guarded(torch, rows * r), Guarded(torch, r), Guarded(torch, r * r)
    _lib.check(lib.nncp_normalize_from_gram(_lib.ptr(hhat.view), _lib.ptr(graw), rows, r, _lib.ptr(owned2.view),
                                            _lib.ptr(lam2.view), _lib.ptr(g2.view), st))
    assert owned2.intact() and lam2.intact() and g2.intact()
    assert rel_fro(owned2.view.cpu().numpy().reshape(rows, r), hn) <= 1e-12
    assert rel_fro(g2.view.cpu().numpy().reshape(r, r), hn.T @ hn) <= 1e-12
    assert rel_fro(lam2.view.cpu().numpy(), w) <= 1e-12


@pytest.mark.parametrize("order,nranks,me", [(3, 1, 0), (4, 8, 5), (3, 64, 63)])
def test_gamma_publish_guard_bands(env, order, nranks, me):
    P, _lib, torch = env
    lib = _lib.load()
    r = 7
    rng = np.random.default_rng(order * nranks)
    g = np.stack([(lambda a: a.T @ a)(rng.random((9, r))) for _ in range(order)])
    lam = rng.random(r)
    status = torch.zeros((order, _lib.STATUS_WORDS), dtype=torch.int32, device="cuda")
    _lib.check(lib.nncp_status_reset_n(_lib.ptr(status), order, _lib.stream_handle()))
    status[1, 3] = 1
    status[1, 2] = 12345
    status[0, 0] = 5
    codes, gamma = Guarded(torch, nranks * order, fill=3.0), Guarded(torch, 1)
    masks = torch.full((2 * order + 8,), -7, dtype=torch.int32, device="cuda")
    dg, dl = torch.as_tensor(g, device="cuda"), torch.as_tensor(lam, device="cuda")   # alive across the launch
    _lib.check(lib.nncp_gamma_publish(_lib.ptr(dg), order, r, _lib.ptr(dl), _lib.ptr(gamma.view),
                                      _lib.ptr(status), order, _lib.ptr(codes.view), nranks * order, me * order,
                                      _lib.ptr(masks), _lib.stream_handle()))
    assert codes.intact() and gamma.intact()
    c = codes.view.cpu().numpy()
    want = np.zeros(nranks * order)
    want[me * order + 1] = 2.0 ** 32 + 12345
    assert np.array_equal(c, want)
    mk = masks.cpu().numpy()
    assert mk[0] == 5 and np.all(mk[2 * order:] == -7)
    st = status.cpu().numpy()
    assert np.all(st[:, 3] == 0) and np.all(st[:, 2] == 2**31 - 1) and np.all(st[:, 0] == 0)   # reset
    gamma_ref = float(lam @ (np.prod(g, axis=0) @ lam))
    assert abs(gamma.view.item() - gamma_ref) <= 1e-12 * abs(gamma_ref)


def test_khatri_rao_guard_bands(env):
    P, _lib, torch = env
    lib = _lib.load()
    rng = np.random.default_rng(4)
    fs = [rng.random((d, 3)) for d in (5, 1, 7, 2)]
    n = 5 * 7 * 2 * 3
    out = Guarded(torch, n)
    dev = [torch.as_tensor(f, device="cuda") for f in fs]
    _lib.check(lib.nncp_khatri_rao(_lib.ptrs(dev), _lib.i64([5, 1, 7, 2]), 4, 3, _lib.ptr(out.view),
                                   _lib.stream_handle()))
    assert out.intact()
    assert np.array_equal(out.view.cpu().numpy().reshape(-1, 3), O.khatri_rao(fs))
