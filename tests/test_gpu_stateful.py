"""UCP / ADMM / NES on the device vs the live reference's golden vectors."""

import warnings

import numpy as np
import pytest

from oracle import nncp_oracle as O
from tests.conftest import rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as pkg

    return pkg


def _np(t):
    return t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)


def test_updates_vs_golden(P, golden):
    g = golden("stateful.npz")
    for k in range(int(g["nst"])):
        s, m, cur = g[f"s{k}_s"], g[f"s{k}_m"], g[f"s{k}_cur"]
        inp = P.UpdateInputs(s, m, cur)
        assert rel_fro(_np(P.ucp_update(inp)), g[f"s{k}_ucp"]) <= 1e-10, k
        st = P.UpdaterState()
        x1 = _np(P.admm_update(inp, st))
        assert st.last_inner_iters == int(g[f"s{k}_admm1_iters"]), k
        assert rel_fro(x1, g[f"s{k}_admm1"]) <= 1e-9, k
        x2 = _np(P.admm_update(P.UpdateInputs(s, m, x1), st))
        assert rel_fro(x2, g[f"s{k}_admm2"]) <= 1e-9, k
        assert rel_fro(_np(st.admm_dual), g[f"s{k}_admm_dual"]) <= 1e-8, k
        nst = P.UpdaterState()
        xn = _np(P.nesterov_update(inp, nst))
        assert nst.last_inner_iters == int(g[f"s{k}_nes_iters"]), k
        assert rel_fro(xn, g[f"s{k}_nes"]) <= 1e-9, k
        from paper_1909_01149_b200.updaters import nesterov_hyperparams

        hyp = np.array(nesterov_hyperparams(s))
        ref = g[f"s{k}_hyper"]
        assert np.allclose(hyp, ref, rtol=1e-9, atol=1e-12), (k, hyp, ref)


def test_known_answers(P):
    # test_updaters.py:202-208 ADMM scalar one step
    st = P.UpdaterState()
    from paper_1909_01149_b200.updaters import admm_update, default_admm_rho, nesterov_hyperparams

    out = admm_update(P.UpdateInputs(np.array([[1.0]]), np.array([[-1.0]]), np.zeros((1, 1))), st, rho=1.0,
                      max_steps=1)
    assert np.allclose(_np(out), [[0.0]]) and np.allclose(_np(st.admm_dual), [[0.5]])
    assert default_admm_rho(np.diag([5.0, 3.0])) == 4.0
    # test_updaters.py:268-272 scalar NES optimum
    nst = P.UpdaterState()
    out = P.nesterov_update(P.UpdateInputs(np.array([[1.0]]), np.array([[2.0]]), np.zeros((1, 1))), nst)
    assert np.allclose(_np(out), [[2.0]]) and nst.last_inner_iters <= 3
    # nonpositive rhs stays zero (test_updaters.py:285-288)
    out = P.nesterov_update(P.UpdateInputs(np.eye(2), np.array([[-1.0, -2.0]]), np.zeros((1, 2))),
                            P.UpdaterState())
    assert np.array_equal(_np(out), np.zeros((1, 2)))
    lam, alpha, beta = nesterov_hyperparams(np.eye(3))
    assert lam == 0.0 and abs(alpha - 1.0) < 1e-15 and abs(beta) < 1e-15
    # inner caps (test_acceptance.py:320-343)
    rng = np.random.default_rng(111)
    q, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    s = q @ np.diag(np.logspace(0, 10, 8)) @ q.T
    s = 0.5 * (s + s.T)
    m = rng.standard_normal((6, 8)) * 1e3
    st = P.UpdaterState()
    admm_update(P.UpdateInputs(s, m, np.abs(m)), st)
    assert st.last_inner_iters == 5
    nst = P.UpdaterState()
    P.nesterov_update(P.UpdateInputs(s, m, np.abs(m)), nst)
    assert nst.last_inner_iters == 20
    # UCP singular Gram warns and solves (test_updaters.py:57-62)
    with pytest.warns(UserWarning):
        out = P.ucp_update(P.UpdateInputs(np.array([[1.0, 1.0], [1.0, 1.0]]), np.array([[2.0, 2.0]]),
                                          np.zeros((1, 2))))
    assert np.allclose(_np(out) @ np.array([[1.0, 1.0], [1.0, 1.0]]), [[2.0, 2.0]], atol=1e-6)


def test_runs_vs_golden(P, golden):
    g = golden("stateful.npz")
    for name in [str(n) for n in g["runs"]]:
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        algo = str(g[f"{name}_algo"])
        x = P.DenseTensor(dims, g[f"{name}_x"])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = P.nncp_sequential(x, P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed))
        ref = g[f"{name}_errors"]
        # north-star tolerances for every rule, NES included: its inner step counts and outer
        # acceptance decisions match the reference call for call (tools/nes_probe.py), and the
        # measured gaps are ~1e-14 (profiles/r02_nes_gaps.log)
        trace_tol, fac_tol = 1e-9, 1e-6
        assert len(rep.errors) == len(ref), name
        assert np.max(np.abs(np.array(rep.errors) - ref)) <= trace_tol, (name, np.array(rep.errors) - ref)
        for n in range(len(dims)):
            assert np.max(np.abs(rep.model.factors[n] - g[f"{name}_f{n}"])) <= fac_tol, (name, n)
        assert rel_fro(rep.model.lam, g[f"{name}_lam"]) <= fac_tol
        assert rep.tree_partial_calls == int(g[f"{name}_partials"]), name
        if f"{name}_grid_errors" in g:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                par = P.nncp_parallel(x, P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed,
                                                     grid=(2, 2, 1)))
            assert np.max(np.abs(np.array(par.errors) - g[f"{name}_grid_errors"])) <= trace_tol, name
            calls = [par.counters.calls.get(c, 0) for c in ("ReduceScatter", "AllGather", "AllReduce")]
            assert calls == list(g[f"{name}_grid_calls"]), (name, calls)


@pytest.mark.parametrize("algo", ["ucp", "mu", "hals", "bpp", "admm", "nes"])
def test_uneven_dims_and_blocks_all_algorithms(P, algo):
    """test_driver.py:227-236: sequential == (2,2,1) grid for every update rule."""
    x, _ = P.generate_synthetic(P.SyntheticSpec((7, 5, 6), 2, seed=12))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        seq = P.nncp_sequential(x, P.RunConfig(rank=2, algorithm=algo, max_iters=6, tol=0.0, seed=5))
        par = P.nncp_parallel(x, P.RunConfig(rank=2, algorithm=algo, max_iters=6, tol=0.0, seed=5, grid=(2, 2, 1)))
    tol = 1e-10
    assert np.allclose(seq.errors, par.errors, rtol=0, atol=tol)
    for a, b in zip(seq.model.factors, par.model.factors):
        assert np.allclose(a, b, rtol=0, atol=max(tol, 1e-10) * 100)


@pytest.mark.parametrize("algo", ["admm", "nes"])
def test_inner_runner_uses_call_rows_not_capacity(P, algo):
    """A grid rank's runner is sized for its largest owned block; a call with fewer rows
    must touch only those rows (regression: the launch used the capacity, read past the
    smaller operands and let stale memory into the stopping test)."""
    import torch
    from paper_1909_01149_b200.tensor_ops import Workspace
    from paper_1909_01149_b200.updaters import AdmmRunner, NesterovRunner, _SPack, local_reduce

    rng = np.random.default_rng(3)
    r, rows, cap = 4, 3, 11
    a = rng.random((9, r))
    s = torch.tensor(a.T @ a, dtype=torch.float64, device="cuda")
    dev = dict(dtype=torch.float64, device="cuda")
    m_np = rng.random((rows, r))
    res = []
    for capacity in (rows, cap):
        # operands are views into NaN-filled buffers with room behind them
        back = [torch.full((cap, r), float("nan"), **dev) for _ in range(3)]
        m, cur, aux = (b[:rows] for b in back)
        m.copy_(torch.tensor(m_np, **dev))
        cur.copy_(m * 0.5)
        if algo == "admm":
            aux.zero_()
        else:
            aux.copy_(cur)
        runner = (AdmmRunner if algo == "admm" else NesterovRunner)(capacity, r, torch.device("cuda"),
                                                                   Workspace(1 << 20))
        for buf in (runner.buf if algo == "admm" else runner.x + runner.y):
            buf.fill_(float("nan"))
        x, steps = runner.run(_SPack.explicit(s), m, cur, aux, local_reduce)
        res.append((x[:rows].cpu().numpy(), steps))
    assert np.isfinite(res[0][0]).all()
    assert np.array_equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]


def test_ucp_lstsq_fallback_matches_reference(P):
    """S singular even with the ridge (indefinite or zero): the reference's minimum-norm
    np.linalg.lstsq(S, M^T, rcond=None) (updaters.py:87-88), now on the device (Jacobi
    eigendecomposition + pseudo-inverse) instead of NotImplementedError."""
    rng = np.random.default_rng(12)
    q, _ = np.linalg.qr(rng.standard_normal((5, 5)))
    cases = [np.diag([2.0, -1.0, 0.0]),                         # indefinite with a zero eigenvalue
             np.zeros((4, 4)),                                   # zero Gram: lstsq gives 0
             q @ np.diag([3.0, 1.0, -0.5, 0.0, 0.0]) @ q.T]      # rotated, rank 3, indefinite
    for s in cases:
        s = 0.5 * (s + s.T)
        m = rng.standard_normal((9, s.shape[0]))
        with pytest.warns(UserWarning, match="ridge"):
            got = _np(P.ucp_update(P.UpdateInputs(s, m, np.zeros_like(m))))
        with pytest.warns(UserWarning, match="ridge"):
            want = O.ucp_update(s, m)
        assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want))), s
