"""BPP's S and S^-1 formed ahead of the update on another stream (nncp_bpp_prepare,
DESIGN.md §4.3): the update that finds the prepared block must return exactly what it
returns when it forms S and S^-1 itself (the same elimination), use a block at most
once, and ignore a block prepared for another mode."""

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


def _problem(order, r, rows, seed):
    rng = np.random.default_rng(seed)
    hs = [rng.random((96, r)) for _ in range(order)]
    hs = [h / np.linalg.norm(h, axis=0) for h in hs]
    g = np.stack([h.T @ h for h in hs])
    xtrue = np.maximum(rng.standard_normal((rows, r)) + 0.8, 0.0)
    s = np.prod(g[1:], axis=0)
    m = xtrue @ s - np.where(xtrue > 0.0, 0.0, rng.random((rows, r)) + 0.1)
    return g, m


def _update(env, g, m, order, mode, r, sets, prepare_mode=None):
    torch, _lib, lib = env
    rows = m.shape[0]
    dg, dm = torch.as_tensor(g, device="cuda"), torch.as_tensor(m, device="cuda")
    cur = torch.zeros_like(dm)
    out = torch.empty_like(dm)
    nsq = torch.empty(r, dtype=torch.float64, device="cuda")
    status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device="cuda")
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    st = _lib.stream_handle()
    _lib.check(lib.nncp_status_reset(_lib.ptr(status), st))
    if prepare_mode is not None:
        side = torch.cuda.Stream()
        fork = torch.cuda.Event()
        fork.record()
        side.wait_event(fork)
        with torch.cuda.stream(side):
            _lib.check(lib.nncp_bpp_prepare(_lib.ptr(dg), order, prepare_mode, r, _lib.ptr(sets), rows,
                                            _lib.stream_handle()))
        done = torch.cuda.Event()
        done.record(side)
        torch.cuda.current_stream().wait_event(done)
    _lib.check(lib.nncp_update_ex(3, _lib.ptr(dg), order, mode, r, _lib.ptr(dm), _lib.ptr(cur), None, rows,
                                  _lib.ptr(out), _lib.ptr(nsq), None, _lib.ptr(status), 1e-16, _lib.ptr(sets), 0,
                                  _lib.vp(ws.data_ptr()), ws.numel(), st))
    torch.cuda.synchronize()
    return out.cpu().numpy(), nsq.cpu().numpy(), status.cpu().numpy()


@pytest.mark.parametrize("order,r,rows", [(3, 5, 300), (3, 16, 257), (4, 32, 256), (4, 64, 130), (3, 32, 1)])
def test_prepared_inverse_is_bitwise_the_update_own(env, order, r, rows):
    torch, _lib, lib = env
    g, m = _problem(order, r, rows, order * 100 + r)
    words = int(lib.nncp_bpp_sets_words(rows, r))
    off = (rows + 1) // 2 * 2
    assert words >= off + 4 + 2 * r * r
    for mode in range(order):
        for warm in (False, True):
            base = torch.zeros(words, dtype=torch.int64, device="cuda")
            if warm:   # a warm start from the cold run's final sets
                _update(env, g, m, order, mode, r, base)
            sets_a, sets_b = base.clone(), base.clone()
            out_a, nsq_a, st_a = _update(env, g, m, order, mode, r, sets_a)
            out_b, nsq_b, st_b = _update(env, g, m, order, mode, r, sets_b, prepare_mode=mode)
            assert np.array_equal(out_a, out_b), (mode, warm, float(np.max(np.abs(out_a - out_b))))
            assert np.array_equal(nsq_a, nsq_b)
            assert np.array_equal(st_a, st_b)
            assert torch.equal(sets_a[:rows], sets_b[:rows])
            assert int(sets_b[off].item()) == 0           # the block was used, and only once


def test_block_for_another_mode_is_ignored(env):
    torch, _lib, lib = env
    order, r, rows = 3, 16, 200
    g, m = _problem(order, r, rows, 7)
    words = int(lib.nncp_bpp_sets_words(rows, r))
    off = (rows + 1) // 2 * 2
    sets_a = torch.zeros(words, dtype=torch.int64, device="cuda")
    sets_b = torch.zeros(words, dtype=torch.int64, device="cuda")
    out_a, nsq_a, _ = _update(env, g, m, order, 2, r, sets_a)
    out_b, nsq_b, _ = _update(env, g, m, order, 2, r, sets_b, prepare_mode=0)   # S of mode 0: not mode 2's
    assert np.array_equal(out_a, out_b) and np.array_equal(nsq_a, nsq_b)
    assert int(sets_b[off].item()) != 0                   # left for a mode-0 update


@pytest.mark.parametrize("graph", [None, False])
@pytest.mark.parametrize("dims", [(24, 20, 16, 18), (160, 120, 20, 18)])   # fused update tail / separate kernels
def test_sweeps_with_prepared_inverse_equal_in_update_bitwise(env, graph, dims):
    """Whole BPP runs (4-way, graph replays or eager sweeps): the side-stream S / S^-1 fork
    and join change nothing in the result."""
    import os

    import paper_1909_01149_b200 as P

    rng = np.random.default_rng(11)
    r = 12
    hs = [rng.random((d, r)) for d in dims]
    from oracle import nncp_oracle as O

    x = O.khatri_rao(hs) @ np.ones(r)
    x = x + 0.02 * np.sqrt(np.mean(x * x)) * np.abs(rng.standard_normal(x.size))
    reps = []
    for flag in ("0", "1"):
        os.environ["NNCP_BPP_PREPARE"] = flag
        try:
            reps.append(P.nncp_sequential(P.DenseTensor(dims, x), P.RunConfig(
                rank=r, algorithm="bpp", max_iters=6, tol=0.0, cuda_graph=graph, mttkrp_kernel="fp64")))
        finally:
            os.environ.pop("NNCP_BPP_PREPARE", None)
    a, b = reps
    assert a.errors == b.errors
    for fa, fb in zip(a.model.factors, b.model.factors):
        assert np.array_equal(fa, fb)
    assert np.array_equal(a.model.lam, b.model.lam)
