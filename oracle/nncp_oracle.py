"""CPU oracle for the dense NNCP hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's algorithm
(`/root/reference/pkg/src/nncp`, pure Python + numpy/OpenBLAS) for the one
path this repository accelerates: dimension-tree MTTKRP, Gram/Hadamard
normal equations, the MU / HALS / ANLS-BPP factor updates (plus UCP, ADMM and
Nesterov with outer extrapolation, the widened rows), column normalisation
and the Gram-trick relative error.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it, and only as the checker or the
timed CPU baseline ("port").  The product path (``paper_1909_01149_b200``)
never imports this file.

Parity pin: every function here is checked against golden vectors produced
by importing the live reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and against the
reference tests' hand-computed known answers (``tests/test_oracle.py``).

Layout conventions follow the reference (`tensor_ops.py:1-13`): a tensor is
a flat float64 buffer with the mode-1 index fastest; factor matrices are
row-major (I_n, R); Khatri-Rao rows are linearised with the FIRST listed
factor fastest.
"""

from __future__ import annotations

import math
import warnings

import numpy as np

MU_EPSILON = 1e-16          # updaters.py:27
BPP_BACKUP_TRIES = 3        # updaters.py:28


# ---------------------------------------------------------------------------
# tensor primitives (tensor_ops.py)
# ---------------------------------------------------------------------------

def unfold_leading(data: np.ndarray, dims, split: int) -> np.ndarray:
    """X_(1:S) as a zero-copy column-major matrix (tensor_ops.py:64-74)."""
    rows = int(np.prod(dims[:split]))
    return data.reshape((rows, -1), order="F")


def khatri_rao(factors) -> np.ndarray:
    """Row (i_1..i_m) = prod_j H_j(i_j, :), first factor fastest (tensor_ops.py:121-137)."""
    acc = np.asarray(factors[0], dtype=np.float64)
    for h in factors[1:]:
        h = np.asarray(h, dtype=np.float64)
        # new index slower than everything accumulated so far
        acc = np.einsum("jr,ir->jir", h, acc).reshape(-1, acc.shape[1])
    return acc


def gram(h: np.ndarray) -> np.ndarray:
    """Symmetrised H^T H (tensor_ops.py:140-143, driver.py:351-353)."""
    g = h.T @ h
    return 0.5 * (g + g.T)


def hadamard_excluding(grams, exclude: int) -> np.ndarray:
    """Elementwise product of all Grams but one (tensor_ops.py:146-155)."""
    out = np.ones_like(grams[0])
    for m, g in enumerate(grams):
        if m != exclude:
            out = out * g
    return out


def naive_mttkrp(data: np.ndarray, dims, factors, mode: int) -> np.ndarray:
    """Direct einsum MTTKRP (tensor_ops.py:158-185)."""
    n = len(dims)
    arr = data.reshape(dims, order="F")
    letters = "abcdefghijklm"
    terms, ops = [letters[:n]], [arr]
    for m in range(n):
        if m != mode:
            terms.append(letters[m] + "z")
            ops.append(factors[m])
    return np.einsum(",".join(terms) + "->" + letters[mode] + "z", *ops, optimize=True)


def normalize_columns(h: np.ndarray):
    """(tensor_ops.py:198-205)."""
    w = np.sqrt(np.sum(h * h, axis=0))
    return h / np.where(w > 0.0, w, 1.0), w


# ---------------------------------------------------------------------------
# dimension tree (dimtree.py)
# ---------------------------------------------------------------------------

def choose_split(dims, strict: bool = False) -> int:
    """Smallest S with prod(dims[:S]) >= prod(dims[S:]) (dimtree.py:25-39)."""
    n = len(dims)
    for s in range(1, n):
        left, right = int(np.prod(dims[:s])), int(np.prod(dims[s:]))
        if left > right or (not strict and left == right):
            return s
    return n - 1


def partial_left(data, dims, split, factors) -> np.ndarray:
    """T_L = X_(1:S) . KRP(H_{S+1..N}); returned flat, rank slowest (dimtree.py:111-117,127)."""
    t = unfold_leading(data, dims, split) @ khatri_rao(factors[split:])
    return t.ravel(order="F")


def partial_right(data, dims, split, factors) -> np.ndarray:
    """T_R = X_(1:S)^T . KRP(H_{1..S}) (dimtree.py:118-124,127)."""
    t = unfold_leading(data, dims, split).T @ khatri_rao(factors[:split])
    return t.ravel(order="F")


def ttv_trailing(temp, lead: int, rank: int, coeff) -> np.ndarray:
    """out[l, r] = sum_j T_r[l, j] coeff[j, r] (dimtree.py:159-165); flat rank slowest."""
    t = temp.reshape((lead, -1, rank), order="F")
    out = np.empty((lead, rank), order="F")
    for r in range(rank):  # one BLAS matvec per rank block, as the reference
        out[:, r] = t[:, :, r] @ coeff[:, r]
    return out.ravel(order="F")


def ttv_leading(temp, lead: int, rank: int, coeff) -> np.ndarray:
    """out[j, r] = sum_l T_r[l, j] coeff[l, r] (dimtree.py:166-172); flat rank slowest."""
    t = temp.reshape((lead, -1, rank), order="F")
    out = np.empty((t.shape[1], rank), order="F")
    for r in range(rank):
        out[:, r] = t[:, :, r].T @ coeff[:, r]
    return out.ravel(order="F")


class DimTree:
    """Sweep state machine of dimtree.py:183-302 (ascending modes, two partials/sweep)."""

    def __init__(self, dims, rank, strict=False):
        self.dims = tuple(int(d) for d in dims)
        self.rank = int(rank)
        self.split = choose_split(self.dims, strict)
        self.partial_calls = 0
        self._left = self._right = None
        self._expected = None

    def begin_iteration(self):
        self._left = self._right = None
        self._expected = 0

    def _as_rows(self, flat, rows):
        return np.ascontiguousarray(flat.reshape((rows, self.rank), order="F"))

    def mttkrp(self, data, factors, mode):
        d, s, n, r = self.dims, self.split, len(self.dims), self.rank
        if self._expected is None or mode != self._expected:
            raise RuntimeError("modes must be requested in ascending order after begin_iteration")
        if mode == 0:
            self.partial_calls += 1
            root = partial_left(data, d, s, factors)
            if s == 1:
                res = root
            else:
                self._left = (root, d[:s])
                res = ttv_trailing(root, d[0], r, khatri_rao(factors[1:s]))
        elif mode < s:
            temp, ret = self._left
            if mode < s - 1:
                temp = ttv_leading(temp, ret[0], r, factors[mode - 1])
                ret = ret[1:]
                self._left = (temp, ret)
                res = ttv_trailing(temp, ret[0], r, khatri_rao(factors[mode + 1:s]))
            else:
                res = ttv_leading(temp, ret[0], r, factors[mode - 1])
                self._left = None
        elif mode == s:
            self.partial_calls += 1
            root = partial_right(data, d, s, factors)
            if s == n - 1:
                res = root
            else:
                self._right = (root, d[s:])
                res = ttv_trailing(root, d[s], r, khatri_rao(factors[s + 1:]))
        else:
            temp, ret = self._right
            if mode < n - 1:
                temp = ttv_leading(temp, ret[0], r, factors[mode - 1])
                ret = ret[1:]
                self._right = (temp, ret)
                res = ttv_trailing(temp, ret[0], r, khatri_rao(factors[mode + 1:]))
            else:
                res = ttv_leading(temp, ret[0], r, factors[mode - 1])
                self._right = None
        self._expected = mode + 1 if mode + 1 < n else None
        return self._as_rows(res, d[mode])

    def mttkrp_last_mode(self, data, factors):
        """One right partial + leading chain (dimtree.py:289-302)."""
        d, s, n, r = self.dims, self.split, len(self.dims), self.rank
        self.partial_calls += 1
        temp, ret = partial_right(data, d, s, factors), d[s:]
        for m in range(s, n - 1):
            temp = ttv_leading(temp, ret[0], r, factors[m])
            ret = ret[1:]
        return self._as_rows(temp, d[n - 1])


# ---------------------------------------------------------------------------
# NNLS updates (updaters.py)
# ---------------------------------------------------------------------------

class BppCycling(RuntimeError):
    def __init__(self, row):
        super().__init__(f"block principal pivoting cycled on column {row}")
        self.column = row


def mu_update(s, m, cur):
    """H * M / (H S + eps) (updaters.py:91-94)."""
    return cur * m / (cur @ s + MU_EPSILON)


def hals_update(s, m, cur):
    """Gauss-Seidel column sweep, clamp at zero, skip s_rr <= 0 (updaters.py:97-118)."""
    h = cur.copy()
    for r in range(s.shape[0]):
        d = s[r, r]
        if d <= 0.0:
            warnings.warn(f"zero gram diagonal in column {r}, skipping")
            continue
        col = h[:, r] + (m[:, r] - h @ s[:, r]) / d
        h[:, r] = np.maximum(col, 0.0)
    return h


def bpp_row(s, f, row):
    """Block principal pivoting for min_{x>=0} .5x'Sx - f'x (updaters.py:121-155)."""
    r = s.shape[0]
    passive = np.zeros(r, dtype=bool)
    x = np.zeros(r)
    y = -f.copy()
    best = r + 1
    backup = BPP_BACKUP_TRIES
    for _ in range(5 * r + 1):
        viol = (passive & (x < 0)) | (~passive & (y < 0))
        k = int(viol.sum())
        if k == 0:
            return x
        if k < best:
            best, backup = k, BPP_BACKUP_TRIES
            passive = passive ^ viol
        elif backup > 0:
            backup -= 1
            passive = passive ^ viol
        else:
            j = int(np.flatnonzero(viol)[-1])
            passive[j] = not passive[j]
        x = np.zeros(r)
        y = np.zeros(r)
        if passive.any():
            x[passive] = np.linalg.solve(s[np.ix_(passive, passive)], f[passive])
        if not passive.all():
            y[~passive] = s[~passive][:, passive] @ x[passive] - f[~passive]
    raise BppCycling(row)


def bpp_update(s, m, cur=None):
    """(updaters.py:158-164)."""
    out = np.empty_like(m)
    for i in range(m.shape[0]):
        out[i] = bpp_row(s, m[i], i)
    return out


ADMM_INNER_CAP = 5          # updaters.py:25
NESTEROV_INNER_CAP = 20     # updaters.py:26


def ucp_update(s, m, cur=None):
    """Unconstrained Cholesky solve with the ridge fallback (updaters.py:77-88)."""
    from scipy.linalg import LinAlgError, cho_factor, cho_solve

    try:
        return cho_solve(cho_factor(s), m.T).T
    except LinAlgError:
        warnings.warn("singular gram in unconstrained update, adding ridge")
        ridge = 1e-12 * np.trace(s) / s.shape[0]
        try:
            return cho_solve(cho_factor(s + ridge * np.eye(s.shape[0])), m.T).T
        except LinAlgError:
            return np.linalg.lstsq(s, m.T, rcond=None)[0].T


def admm_update(s, m, cur, dual, rho=None, max_steps=ADMM_INNER_CAP, rtol=1e-4, reduce=lambda v: v):
    """Three-step ADMM splitting, returns (x, dual, steps) (updaters.py:167-220)."""
    from scipy.linalg import cho_factor, cho_solve

    r = s.shape[0]
    if rho is None:
        rho = float(np.trace(s)) / r
        rho = rho if rho > 0.0 else 1.0
    chol = cho_factor(s + rho * np.eye(r))
    x = cur
    u = np.zeros_like(cur) if dual is None else dual
    steps = 0
    for _ in range(max_steps):
        xhat = cho_solve(chol, (m + rho * (x + u)).T).T
        xprev = x
        x = np.maximum(xhat - u, 0.0)
        u = u + x - xhat
        steps += 1
        sq = reduce(np.array([np.sum((x - xhat) ** 2), np.sum(x ** 2), np.sum(xhat ** 2),
                              np.sum((x - xprev) ** 2), np.sum(u ** 2)]))
        gap, nx, nxhat, step, nu = np.sqrt(sq)
        if gap <= rtol * max(nx, nxhat) and rho * step <= rtol * nu * rho:
            break
    return x, u, steps


def nesterov_hyperparams(s, prox_floor=1e-6):
    """(lam, alpha, beta) from the Gram spectrum (updaters.py:223-243)."""
    ev = np.linalg.eigvalsh(s)
    big, small = float(ev[-1]), max(float(ev[0]), 0.0)
    if big <= 0.0:
        lam = 1.0
    elif small / big >= prox_floor:
        lam = 0.0
    else:
        lam = (prox_floor * big - small) / (1.0 - prox_floor)
    q = (small + lam) / (big + lam)
    return lam, 1.0 / (big + lam), (1.0 - np.sqrt(q)) / (1.0 + np.sqrt(q))


def nesterov_update(s, m, cur, xstar, max_iters=NESTEROV_INNER_CAP, tol=1e-8, reduce=lambda v: v):
    """Accelerated projected gradient with proximal centre (updaters.py:250-281); returns (x, steps)."""
    lam, alpha, beta = nesterov_hyperparams(s)
    xstar = cur if xstar is None else xstar
    x = y = cur
    steps = 0
    for _ in range(max_iters):
        grad = y @ s - m + lam * (y - xstar)
        xn = np.maximum(y - alpha * grad, 0.0)
        steps += 1
        dmax, xmax = reduce(np.array([np.max(np.abs(xn - x)) if xn.size else 0.0,
                                      np.max(np.abs(xn)) if xn.size else 0.0]))
        y = xn + beta * (xn - x)
        x = xn
        if dmax <= tol * (1.0 + xmax):
            break
    return x, steps


UPDATERS = {"mu": lambda s, m, c: mu_update(s, m, c),
            "ucp": lambda s, m, c: ucp_update(s, m, c),
            "hals": lambda s, m, c: hals_update(s, m, c),
            "bpp": lambda s, m, c: bpp_update(s, m, c)}


# ---------------------------------------------------------------------------
# driver (driver.py)
# ---------------------------------------------------------------------------

def init_factor(seed: int, mode: int, rows: int, rank: int) -> np.ndarray:
    """Philox keyed by (seed, mode), entry (i, r) = draw i*R + r (driver.py:137-143)."""
    key = np.array([seed, mode], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).random((rows, rank))


def eps_from_terms(alpha, beta, gamma) -> float:
    """(driver.py:146-148)."""
    return float(np.sqrt(max(0.0, alpha - 2.0 * beta + gamma) / alpha))


def run_sequential(data, dims, rank, algorithm="bpp", max_iters=100, tol=1e-6, seed=0,
                   use_dimtree=True, strict_split=False, initial_factors=None,
                   initial_lam=None, timings=None, init_error="naive"):
    """Alternating-update NNCP, sequential runtime (driver.py:331-449, 495-505).

    Returns (errors, factors, lam, split, partial_calls).  ``timings``, when a
    list, receives the wall seconds of every row (row 0 = initialisation).
    """
    import time

    dims = tuple(int(d) for d in dims)
    order = len(dims)
    data = np.ascontiguousarray(data, dtype=np.float64).ravel()
    upd = UPDATERS.get(algorithm)
    t0 = time.perf_counter()
    alpha = float(np.dot(data, data))
    if alpha <= 0.0:
        raise ValueError("zero tensor has no relative error")
    if initial_factors is not None:
        hs = [np.array(h, dtype=np.float64) for h in initial_factors]
        lam = np.array(initial_lam, dtype=np.float64) if initial_lam is not None else np.ones(rank)
    else:
        hs = [init_factor(seed, n, dims[n], rank) for n in range(order)]
        lam = np.ones(rank)
    grams = [gram(h) for h in hs]
    tree = DimTree(dims, rank, strict_split) if use_dimtree else None
    duals = [None] * order          # ADMM state per mode (updaters.py:56-68)
    centres = [None] * order        # Nesterov proximal centre per mode
    if init_error == "none":   # bench baseline only: the init row is not timed, skip its MTTKRP
        errors = [float("nan")]
    else:
        if init_error == "naive":
            m0 = naive_mttkrp(data, dims, hs, order - 1)
        else:  # same quantity through the tree's last-mode path
            m0 = DimTree(dims, rank, strict_split).mttkrp_last_mode(data, hs)
        beta0 = float(np.dot(m0.ravel(), (hs[-1] * lam).ravel()))
        gamma0 = float(lam @ (np.prod(grams, axis=0) @ lam))
        errors = [eps_from_terms(alpha, beta0, gamma0)]
    if timings is not None:
        timings.append(time.perf_counter() - t0)
    for it in range(1, max_iters + 1):
        t0 = time.perf_counter()
        if algorithm == "nes":
            prev_hs, prev_lam = [h.copy() for h in hs], lam.copy()
        if tree is not None:
            tree.begin_iteration()
        for n in range(order):
            mb = tree.mttkrp(data, hs, n) if tree is not None else naive_mttkrp(data, dims, hs, n)
            s_n = hadamard_excluding(grams, n)
            try:
                if algorithm == "admm":
                    hhat, duals[n], _ = admm_update(s_n, mb, hs[n] * lam, duals[n])
                elif algorithm == "nes":
                    hhat, _ = nesterov_update(s_n, mb, hs[n] * lam, centres[n])
                    centres[n] = hhat.copy()
                else:
                    hhat = upd(s_n, mb, hs[n] * lam)
            except Exception as exc:
                raise RuntimeError(f"NNLS update failed at iteration {it}, mode {n + 1}") from exc
            w = np.sqrt(np.sum(hhat * hhat, axis=0))
            hs[n] = hhat / np.where(w > 0.0, w, 1.0)
            lam = w
            grams[n] = gram(hs[n])
            if n == order - 1:
                m_last, hhat_last, s_last = mb, hhat, s_n
        beta = float(np.dot(m_last.ravel(), hhat_last.ravel()))
        gamma = float(lam @ ((s_last * grams[-1]) @ lam))
        eps = eps_from_terms(alpha, beta, gamma)
        errors.append(eps)
        if algorithm == "nes":
            hs, lam, grams = _nes_accelerate(data, dims, tree, it, eps, alpha, hs, lam, grams, prev_hs,
                                             prev_lam, use_dimtree)
        if timings is not None:
            timings.append(time.perf_counter() - t0)
        if eps <= tol:
            break
    calls = tree.partial_calls if tree is not None else 0
    return errors, hs, lam, (tree.split if tree is not None else None), calls


def _nes_accelerate(data, dims, tree, it, eps, alpha, hs, lam, grams, prev_hs, prev_lam, use_dimtree):
    """Outer extrapolation, accepted only if strictly better (driver.py:452-492, 310-328)."""
    step = float(it) ** (1.0 / len(hs))
    cand = [np.maximum(h + step * (h - hp), 0.0) for h, hp in zip(hs, prev_hs)]
    cand_lam = np.maximum(lam + step * (lam - prev_lam), 0.0)
    if use_dimtree:
        mb = tree.mttkrp_last_mode(data, cand)
    else:
        mb = naive_mttkrp(data, dims, cand, len(dims) - 1)
    beta = float(np.dot(mb.ravel(), (cand[-1] * cand_lam).ravel()))
    cg = [h.T @ h for h in cand]
    gamma = float(cand_lam @ (np.prod(cg, axis=0) @ cand_lam))
    if not eps_from_terms(alpha, beta, gamma) < eps:
        return hs, lam, grams
    w = np.sqrt(np.stack([np.sum(h * h, axis=0) for h in cand]))
    scale = np.where(w > 0.0, w, 1.0)
    new = [h / scale[n] for n, h in enumerate(cand)]
    return new, cand_lam * np.prod(w, axis=0), [gram(h) for h in new]


def reconstruct(factors, lam) -> np.ndarray:
    """Flat mode-1-fastest model tensor (tensor_ops.py:192-195)."""
    return khatri_rao(factors) @ lam


def relative_error_direct(data, factors, lam) -> float:
    return float(np.linalg.norm(data - reconstruct(factors, lam)) / np.linalg.norm(data))


def block_partition(length: int, parts: int):
    """Balanced blocks, first length%parts get one extra (grid.py:25-31); returns offsets."""
    base, extra = divmod(length, parts)
    lens = [base + 1 if k < extra else base for k in range(parts)]
    offs = [0]
    for x in lens:
        offs.append(offs[-1] + x)
    return offs


def mttkrp_flops(dims, rank) -> int:
    """Two partial MTTKRPs per sweep, 2*I*R each (dimtree.py:130-132)."""
    return 4 * math.prod(dims) * rank
