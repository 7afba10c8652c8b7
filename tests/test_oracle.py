"""Pin the CPU oracle (test infrastructure) against the reference.

Two kinds of pins: golden vectors produced by the live reference
(tests/golden/make_golden.py) and the reference tests' own known answers
(pkg/tests/test_tensor_ops.py, test_dimtree.py, test_updaters.py)."""

import warnings

import numpy as np
import pytest

from oracle import nncp_oracle as O
from tests.conftest import rel_fro


def test_known_answers_tensor_ops():
    # test_tensor_ops.py:85-89 (two-factor KRP)
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert np.array_equal(O.khatri_rao([a, b]),
                          np.array([[5.0, 12.0], [15.0, 24.0], [7.0, 16.0], [21.0, 32.0]]))
    # test_tensor_ops.py:121-123 (Gram hand example)
    assert np.array_equal(O.gram(a), np.array([[10.0, 14.0], [14.0, 20.0]]))
    # test_tensor_ops.py:144-149 (Hadamard of Grams)
    g1 = np.array([[2.0, 1.0], [1.0, 2.0]])
    g2 = np.array([[3.0, 0.0], [0.0, 3.0]])
    g3 = np.array([[9.0, 9.0], [9.0, 9.0]])
    assert np.array_equal(O.hadamard_excluding([g1, g2, g3], 2), np.array([[6.0, 0.0], [0.0, 6.0]]))
    # test_tensor_ops.py:170-174 (naive MTTKRP hand example)
    x = np.arange(1.0, 9.0)
    hs = [np.zeros((2, 2)), np.eye(2), np.ones((2, 2))]
    assert np.array_equal(O.naive_mttkrp(x, (2, 2, 2), hs, 0), np.array([[6.0, 10.0], [8.0, 12.0]]))
    # dimension tree on the same example (test_dimtree.py:156-160)
    t = O.DimTree((2, 2, 2), 2)
    t.begin_iteration()
    assert np.allclose(t.mttkrp(x, hs, 0), np.array([[6.0, 10.0], [8.0, 12.0]]))


def test_known_answers_dimtree():
    assert O.choose_split([128, 128, 128]) == 2                      # test_dimtree.py:19-20
    assert O.choose_split([1446680, 69, 25]) == 1
    assert O.choose_split([384] * 4) == 2 and O.choose_split([384] * 4, strict=True) == 3
    assert O.choose_split([5, 3]) == 1 and O.choose_split([3, 5]) == 1
    assert O.choose_split([2, 2, 100]) == 2
    # test_dimtree.py:94-98 hand matvec
    out = O.ttv_trailing(np.array([1.0, 3.0, 2.0, 4.0]), 2, 1, np.ones((2, 1)))
    assert np.array_equal(out, np.array([3.0, 7.0]))


def test_known_answers_updaters():
    assert np.allclose(O.mu_update(np.array([[2.0]]), np.array([[4.0]]), np.array([[1.0]])), 2.0)
    assert np.allclose(O.hals_update(np.array([[2.0]]), np.array([[4.0], [-2.0]]),
                                     np.zeros((2, 1))), [[2.0], [0.0]])
    s = np.array([[1.0, 0.5], [0.5, 1.0]])
    assert np.allclose(O.hals_update(s, np.array([[1.0, 1.0]]), np.zeros((1, 2))), [[1.0, 0.5]])
    with pytest.warns(UserWarning):
        out = O.hals_update(np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([[1.0, 5.0]]),
                            np.array([[0.0, 0.25]]))
    assert np.allclose(out, [[1.0, 0.25]])
    assert np.allclose(O.bpp_update(np.eye(2), np.array([[1.0, 2.0]])), [[1.0, 2.0]])
    assert np.allclose(O.bpp_update(np.array([[1.0]]), np.array([[-3.0]])), [[0.0]])
    assert np.allclose(O.bpp_update(np.array([[2.0, 1.0], [1.0, 2.0]]), np.array([[1.0, -1.0]])),
                       [[0.5, 0.0]], atol=1e-12)
    with pytest.raises(O.BppCycling) as info:
        O.bpp_update(np.array([[1.0, -3.0], [-3.0, 1.0]]), np.array([[0.0, 0.0], [1.0, 1.0]]))
    assert info.value.column == 1


def test_oracle_mttkrp_vs_golden(golden):
    g = golden("mttkrp.npz")
    for k in range(int(g["ncases"])):
        dims = tuple(int(d) for d in g[f"c{k}_dims"])
        r = int(g[f"c{k}_rank"])
        x = g[f"c{k}_x"]
        hs = [g[f"c{k}_h{n}"] for n in range(len(dims))]
        new = [g[f"c{k}_new{n}"] for n in range(len(dims))]
        tree = O.DimTree(dims, r)
        assert tree.split == int(g[f"c{k}_split"])
        tree.begin_iteration()
        cur = [h.copy() for h in hs]
        for n in range(len(dims)):
            got = tree.mttkrp(x, cur, n)
            assert rel_fro(got, g[f"c{k}_m{n}"]) <= 1e-13, (k, n)
            cur[n] = new[n]
        assert tree.partial_calls == 2
        assert rel_fro(O.DimTree(dims, r).mttkrp_last_mode(x, hs), g[f"c{k}_last"]) <= 1e-13
        s = tree.split
        assert rel_fro(O.partial_left(x, dims, s, hs), g[f"c{k}_tl"]) <= 1e-13
        assert rel_fro(O.partial_right(x, dims, s, hs), g[f"c{k}_tr"]) <= 1e-13
        if s >= 2:
            tl = g[f"c{k}_tl"]
            assert rel_fro(O.ttv_trailing(tl, dims[0], r, O.khatri_rao(hs[1:s])),
                           g[f"c{k}_ttv_trail"]) <= 1e-13
            assert rel_fro(O.ttv_leading(tl, dims[0], r, hs[0]), g[f"c{k}_ttv_lead"]) <= 1e-13


def test_oracle_updates_vs_golden(golden):
    g = golden("updates.npz")
    for k in range(int(g["nupd"])):
        s, m, cur = g[f"u{k}_s"], g[f"u{k}_m"], g[f"u{k}_cur"]
        assert rel_fro(O.mu_update(s, m, cur), g[f"u{k}_mu"]) <= 1e-14
        assert rel_fro(O.hals_update(s, m, cur), g[f"u{k}_hals"]) <= 1e-12
        assert np.allclose(O.bpp_update(s, m, cur), g[f"u{k}_bpp"], rtol=1e-10, atol=1e-12)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert np.array_equal(O.hals_update(g["hals_zero_s"], g["hals_zero_m"], g["hals_zero_cur"]),
                              g["hals_zero_out"])


def test_oracle_runs_vs_golden(golden):
    g = golden("runs.npz")
    for name in [str(n) for n in g["names"]]:
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        algo = str(g[f"{name}_algo"])
        errors, hs, lam, split, calls = O.run_sequential(
            g[f"{name}_x"], dims, r, algo, iters, 0.0, iseed)
        assert split == int(g[f"{name}_split"])
        assert calls == 2 * iters
        ref = g[f"{name}_errors"]
        assert len(errors) == len(ref)
        assert np.max(np.abs(np.array(errors) - ref)) <= 1e-12, name
        for n in range(len(dims)):
            assert np.max(np.abs(hs[n] - g[f"{name}_f{n}"])) <= 1e-9, (name, n)
        assert rel_fro(lam, g[f"{name}_lam"]) <= 1e-9


def test_oracle_init_vs_golden(golden):
    g = golden("init.npz")
    for k in range(4):
        seed, mode, rows, rank = (int(v) for v in g[f"i{k}_args"])
        assert np.array_equal(O.init_factor(seed, mode, rows, rank), g[f"i{k}_val"])


def test_error_identity_vs_reconstruction():
    rng = np.random.default_rng(107)
    for _ in range(20):
        dims = tuple(int(d) for d in rng.integers(2, 7, size=3))
        x = rng.random(int(np.prod(dims))) + 0.01
        errors, hs, lam, _, _ = O.run_sequential(x, dims, 2, "hals", 3, 0.0, 1)
        assert abs(errors[-1] - O.relative_error_direct(x, hs, lam)) <= 1e-8


def test_oracle_stateful_vs_golden(golden):
    """UCP / ADMM / NES restatements pinned to the live reference (tests/golden/stateful.npz)."""
    g = golden("stateful.npz")
    for k in range(int(g["nst"])):
        s, m, cur = g[f"s{k}_s"], g[f"s{k}_m"], g[f"s{k}_cur"]
        assert rel_fro(O.ucp_update(s, m), g[f"s{k}_ucp"]) <= 1e-12
        x1, u, steps = O.admm_update(s, m, cur, None)
        assert steps == int(g[f"s{k}_admm1_iters"]) and rel_fro(x1, g[f"s{k}_admm1"]) <= 1e-12
        x2, u, _ = O.admm_update(s, m, x1, u)
        assert rel_fro(x2, g[f"s{k}_admm2"]) <= 1e-12 and rel_fro(u, g[f"s{k}_admm_dual"]) <= 1e-12
        xn, steps = O.nesterov_update(s, m, cur, None)
        assert steps == int(g[f"s{k}_nes_iters"]) and rel_fro(xn, g[f"s{k}_nes"]) <= 1e-12
        assert np.allclose(O.nesterov_hyperparams(s), g[f"s{k}_hyper"], rtol=1e-14, atol=0)
    for name in [str(n) for n in g["runs"]]:
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            errors, hs, lam, _, calls = O.run_sequential(g[f"{name}_x"], dims, r, str(g[f"{name}_algo"]), iters,
                                                         0.0, iseed)
        assert np.max(np.abs(np.array(errors) - g[f"{name}_errors"])) <= 1e-12, name
        assert calls == int(g[f"{name}_partials"]), name
