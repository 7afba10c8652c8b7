"""Per-mode NNLS factor updates on the device (reference: nncp/updaters.py).

Hot path (BASELINE north star): MU (updaters.py:91-94), HALS (97-118) and
ANLS-BPP (121-164) -- one fused kernel each: optional Hadamard-of-Grams
prologue, the row-parallel update, fixed-order column reductions.

Also available (same UpdateInputs boundary): UCP (77-88, one
Cholesky-solve kernel), ADMM (167-220) and the accelerated projected gradient
"NES" (223-281).  ADMM/NES run one launch per inner step; the stopping test of
each step goes through ``hook`` exactly like the reference (sum of five squared
norms / max of two max-abs values), so in a grid run every inner step costs
one All-Reduce, as in the reference.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .tensor_ops import FactorSet, Workspace, as_device, on_host, to_host_if

__all__ = ["UpdateInputs", "UpdaterState", "BppCyclingError", "mu_update", "hals_update", "bpp_update",
           "ucp_update", "admm_update", "nesterov_update", "nesterov_outer_accelerate", "default_admm_rho",
           "nesterov_hyperparams",
           "MU_EPSILON", "BPP_BACKUP_TRIES", "ADMM_INNER_CAP", "NESTEROV_INNER_CAP", "raise_for_status",
           "raise_for_code", "warn_for_status",
           "local_reduce", "AdmmRunner", "NesterovRunner"]

ADMM_INNER_CAP = 5        # updaters.py:25
NESTEROV_INNER_CAP = 20   # updaters.py:26
MU_EPSILON = 1e-16        # updaters.py:27 (compiled into the kernel)
BPP_BACKUP_TRIES = 3      # updaters.py:28 (compiled into the kernel)
NESTEROV_PROX_FLOOR = 1e-6


def local_reduce(value, op: str):
    """Identity reduction for the single-contributor case (updaters.py:31-35)."""
    if op not in ("sum", "min", "max"):
        raise ValueError(f"unknown reduction {op!r}")
    return value


class BppCyclingError(RuntimeError):
    """updaters.py:71-74; ``column`` is the failing factor row."""

    def __init__(self, column: int):
        super().__init__(f"block principal pivoting cycled on column {column}")
        self.column = column


@dataclass
class UpdateInputs:
    """S = A^T A, MTTKRP rows, current rows (updaters.py:38-53); numpy or torch."""

    gram: object
    mttkrp_rows: object
    current: object

    def __post_init__(self):
        r = int(self.gram.shape[0])
        if tuple(self.gram.shape) != (r, r):
            raise ValueError("gram must be square")
        if int(self.mttkrp_rows.shape[1]) != r or int(self.current.shape[1]) != r:
            raise ValueError("rank mismatch between gram and factor rows")
        if int(self.mttkrp_rows.shape[0]) != int(self.current.shape[0]):
            raise ValueError("mttkrp_rows and current must have equal row counts")


@dataclass
class UpdaterState:
    """Per-mode state of the stateful rules (updaters.py:56-68); device tensors here."""

    admm_dual: object = None
    nesterov_prev: object = None
    last_inner_iters: int = 0


def warn_for_status(mask_lo, mask_hi, algo: str = "hals"):
    """The reference's per-update warnings (updaters.py:84,112) from the status mask words."""
    mask = (int(mask_lo) & 0xFFFFFFFF) | ((int(mask_hi) & 0xFFFFFFFF) << 32)
    if algo == "hals" and mask:
        for r in range(64):
            if (mask >> r) & 1:
                warnings.warn(f"zero gram diagonal in column {r}, skipping")
    if algo == "ucp" and mask & 1:
        warnings.warn("singular gram in unconstrained update, adding ridge")


def raise_for_code(kind: int, row: int):
    """The reference's NNLS exceptions (updaters.py:152,163) from a failure kind / row."""
    if kind == 1:
        raise BppCyclingError(int(row))
    if kind == 2:
        raise np.linalg.LinAlgError("Singular matrix")     # what np.linalg.solve raises (updaters.py:152)


def raise_for_status(status_host, algo: str = "hals"):
    """Translate kernel status words into the reference's warnings / exceptions."""
    warn_for_status(status_host[0], status_host[1], algo)
    raise_for_code(int(status_host[3]), int(status_host[2]))


def _run(algo: str, inp: UpdateInputs, mu_eps: float = MU_EPSILON):
    """One device update of every row; numpy out for numpy in (the reference's type)."""
    host = on_host(inp.gram, inp.mttkrp_rows, inp.current)
    lib = _lib.load()
    s = as_device(inp.gram)
    m = as_device(inp.mttkrp_rows)
    cur = as_device(inp.current)
    rows, r = int(m.shape[0]), int(m.shape[1])
    out = torch.empty((rows, r), dtype=torch.float64, device=m.device)
    status = torch.empty(_lib.STATUS_WORDS, dtype=torch.int32, device=m.device)
    ws = Workspace(256 + 8 * ((rows + 3) * (r + 1) + r * r + 4096))
    st = _lib.stream_handle()
    _lib.check(lib.nncp_status_reset(_lib.ptr(status), st))
    _lib.check(lib.nncp_update_ex(_lib.ALGO_CODES[algo], _lib.ptr(s), 0, -1, r, _lib.ptr(m), _lib.ptr(cur), None,
                                  rows, _lib.ptr(out), None, None, _lib.ptr(status), float(mu_eps), None, 0,
                                  ws.ptr, ws.nbytes, st))
    raise_for_status(status.cpu().tolist(), algo)
    return to_host_if(out, host)


def mu_update(inp: UpdateInputs, eps: float = MU_EPSILON):
    """H <- H * M / (H S + eps) (updaters.py:91-94)."""
    return _run("mu", inp, eps)


def hals_update(inp: UpdateInputs, hook=local_reduce):
    """One Gauss-Seidel column sweep (updaters.py:97-118).

    The reference's per-column hook All-Reduce returns a value nobody reads
    (updaters.py:117); the device path does not issue it.
    """
    return _run("hals", inp)


def bpp_update(inp: UpdateInputs):
    """Exact NNLS per row by block principal pivoting (updaters.py:121-164)."""
    return _run("bpp", inp)


def ucp_update(inp: UpdateInputs):
    """Unconstrained Cholesky solve S H^T = M^T with the ridge fallback (updaters.py:77-88)."""
    return _run("ucp", inp)


def default_admm_rho(gram) -> float:
    """rho = trace(S) / R, 1 if not positive (updaters.py:167-170)."""
    g = gram.detach().cpu().numpy() if isinstance(gram, torch.Tensor) else np.asarray(gram, dtype=np.float64)
    rho = float(np.trace(g)) / g.shape[0]
    return rho if rho > 0.0 else 1.0


class _SPack:
    """Where S comes from: (grams stack, order, mode) or an explicit R x R matrix (order 0)."""

    def __init__(self, grams: torch.Tensor, order: int, mode: int):
        self.grams, self.order, self.mode = grams, order, mode

    @classmethod
    def explicit(cls, s):
        return cls(as_device(s), 0, -1)


def _host(t: torch.Tensor):
    return t.detach().cpu().numpy()


def _runner_rows(capacity: int, m: torch.Tensor, *others: torch.Tensor) -> int:
    """Rows of this call: the MTTKRP block's (a grid rank owns a different row count per
    mode; the runner's buffers are sized for the largest).  Launching with the buffer
    capacity would read past the smaller operands."""
    rows = int(m.shape[0])
    if rows > capacity or any(int(t.shape[0]) < rows for t in others):
        raise ValueError(f"inner-solver operands disagree on rows: {rows} (capacity {capacity})")
    return rows


class AdmmRunner:
    """Inner loop of admm_update on device buffers (updaters.py:173-220)."""

    def __init__(self, rows: int, rank: int, device, workspace: Workspace):
        f64 = dict(dtype=torch.float64, device=device)
        self.buf = [torch.empty((rows, rank), **f64), torch.empty((rows, rank), **f64)]
        self.sums = torch.zeros(6, **f64)
        self.status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device=device)
        self.ws = workspace
        self.rows, self.rank = rows, rank

    def run(self, spack: _SPack, m: torch.Tensor, current: torch.Tensor, u: torch.Tensor, hook, rho=None,
            max_steps: int = ADMM_INNER_CAP, rtol: float = 1e-4, status=None, defer_errors: bool = False):
        """``defer_errors``: leave a failed solve in ``status`` instead of raising here, so
        every rank keeps issuing the same hook All-Reduces; the engine raises the same
        error on every rank after the sweep (grid.py:172-203)."""
        lib = _lib.load()
        st = _lib.stream_handle()
        status = self.status if status is None else status
        if rho is not None and rho <= 0.0:
            raise ValueError("rho must be positive")
        rows = _runner_rows(self.rows, m, current, u)
        x = current
        steps = 0
        for k in range(max_steps):
            out = self.buf[k % 2]
            _lib.check(lib.nncp_admm_step(_lib.ptr(spack.grams), spack.order, spack.mode, self.rank,
                                          float(rho) if rho is not None else -1.0, _lib.ptr(m), _lib.ptr(x),
                                          _lib.ptr(u), _lib.ptr(out), rows, _lib.ptr(self.sums),
                                          _lib.ptr(status), self.ws.ptr, self.ws.nbytes, st))
            x = out
            steps += 1
            red = hook(self.sums[:5], "sum")
            host = red.detach().cpu().numpy() if isinstance(red, torch.Tensor) else np.asarray(red)
            rho_used = float(self.sums[5].item())
            if not defer_errors:
                stv = status.cpu().tolist()
                if int(stv[3]):
                    raise_for_status(stv, "admm")
            gap, nx, nxhat, step, nu = np.sqrt(host)
            if gap <= rtol * max(nx, nxhat) and rho_used * step <= rtol * nu * rho_used:
                break
        return x, steps


def _torch_hook(hook):
    """Adapt a reference-style hook (numpy in/out) to device tensors."""
    def run(t: torch.Tensor, op: str):
        res = hook(t.detach().cpu().numpy(), op)
        return np.asarray(res, dtype=np.float64)
    return run


def admm_update(inp: UpdateInputs, state: UpdaterState, hook=local_reduce, rho: float = None,
                max_steps: int = ADMM_INNER_CAP, rtol: float = 1e-4) -> torch.Tensor:
    """Up to ``max_steps`` ADMM rounds, dual persisting in ``state`` (updaters.py:173-220)."""
    host = on_host(inp.gram, inp.mttkrp_rows, inp.current)
    s = as_device(inp.gram)
    m = as_device(inp.mttkrp_rows)
    cur = as_device(inp.current)
    rows, r = int(m.shape[0]), int(m.shape[1])
    u = state.admm_dual
    u = torch.zeros_like(cur) if u is None else as_device(u).clone()
    runner = AdmmRunner(rows, r, m.device, Workspace(256 + 8 * (rows * 6 + 4096)))
    x, steps = runner.run(_SPack.explicit(s), m, cur, u, _torch_hook(hook), rho, max_steps, rtol)
    state.admm_dual = to_host_if(u, host)
    state.last_inner_iters = steps
    return to_host_if(x.clone(), host)


def nesterov_hyperparams(gram, prox_floor: float = NESTEROV_PROX_FLOOR):
    """(lam, alpha, beta) from the extreme eigenvalues of S (updaters.py:223-243), device Jacobi."""
    lib = _lib.load()
    s = as_device(gram)
    hyper = torch.empty(3, dtype=torch.float64, device=s.device)
    _lib.check(lib.nncp_nes_hyper(_lib.ptr(s), 0, -1, int(s.shape[0]), float(prox_floor), _lib.ptr(hyper),
                                  _lib.stream_handle()))
    lam, alpha, beta = hyper.cpu().tolist()
    return lam, alpha, beta


class NesterovRunner:
    """Inner loop of nesterov_update on device buffers (updaters.py:250-281)."""

    def __init__(self, rows: int, rank: int, device, workspace: Workspace):
        f64 = dict(dtype=torch.float64, device=device)
        self.x = [torch.empty((rows, rank), **f64), torch.empty((rows, rank), **f64)]
        self.y = [torch.empty((rows, rank), **f64), torch.empty((rows, rank), **f64)]
        self.maxes = torch.zeros(2, **f64)
        self.hyper = torch.zeros(3, **f64)
        self.ws = workspace
        self.rows, self.rank = rows, rank

    def run(self, spack: _SPack, m: torch.Tensor, current: torch.Tensor, xstar: torch.Tensor, hook,
            max_iters: int = NESTEROV_INNER_CAP, tol: float = 1e-8):
        lib = _lib.load()
        st = _lib.stream_handle()
        rows = _runner_rows(self.rows, m, current, xstar)
        _lib.check(lib.nncp_nes_hyper(_lib.ptr(spack.grams), spack.order, spack.mode, self.rank,
                                      NESTEROV_PROX_FLOOR, _lib.ptr(self.hyper), st))
        x = y = current
        steps = 0
        for k in range(max_iters):
            xo, yo = self.x[k % 2], self.y[k % 2]
            _lib.check(lib.nncp_nes_step(_lib.ptr(spack.grams), spack.order, spack.mode, self.rank,
                                         _lib.ptr(self.hyper), _lib.ptr(m), _lib.ptr(y), _lib.ptr(x),
                                         _lib.ptr(xstar), _lib.ptr(xo), _lib.ptr(yo), rows,
                                         _lib.ptr(self.maxes), self.ws.ptr, self.ws.nbytes, st))
            steps += 1
            red = hook(self.maxes, "max")
            dmax, xmax = (red.detach().cpu().numpy() if isinstance(red, torch.Tensor) else np.asarray(red)).tolist()
            x, y = xo, yo
            if dmax <= tol * (1.0 + xmax):
                break
        return x, steps


def nesterov_update(inp: UpdateInputs, state: UpdaterState, hook=local_reduce,
                    max_iters: int = NESTEROV_INNER_CAP, tol: float = 1e-8) -> torch.Tensor:
    """Accelerated projected gradient with proximal centre state.nesterov_prev (updaters.py:250-281)."""
    host = on_host(inp.gram, inp.mttkrp_rows, inp.current)
    s = as_device(inp.gram)
    m = as_device(inp.mttkrp_rows)
    cur = as_device(inp.current)
    rows, r = int(m.shape[0]), int(m.shape[1])
    xstar = cur if state.nesterov_prev is None else as_device(state.nesterov_prev)
    runner = NesterovRunner(rows, r, m.device, Workspace(256 + 8 * (rows * 3 + 4096)))
    x, steps = runner.run(_SPack.explicit(s), m, cur, xstar, _torch_hook(hook), max_iters, tol)
    out = x.clone()
    state.nesterov_prev = to_host_if(out.clone(), host)
    state.last_inner_iters = steps
    return to_host_if(out, host)


def nesterov_outer_accelerate(model_prev, model_cur, iteration: int, error_fn):
    """Extrapolated candidate H_i + s_i (H_i - H_{i-1}), s_i = i^(1/N), clamped at zero,
    kept only when ``error_fn`` reports a strictly lower error (updaters.py:284-300).
    The extrapolation runs in the device kernel the engine uses (nncp_extrapolate);
    numpy models give numpy candidates."""
    lib = _lib.load()
    host = on_host(model_prev, model_cur)
    step = float(iteration) ** (1.0 / model_cur.order)

    def extrap(cur, prev):
        c, p = as_device(cur), as_device(prev)
        if tuple(c.shape) != tuple(p.shape):
            raise ValueError(f"model shapes differ: {tuple(c.shape)} vs {tuple(p.shape)}")
        out = torch.empty_like(c)
        _lib.check(lib.nncp_extrapolate(_lib.ptr(c), _lib.ptr(p), c.numel(), step, _lib.ptr(out),
                                        _lib.stream_handle()))
        return to_host_if(out, host)

    factors = [extrap(hc, hp) for hp, hc in zip(model_prev.factors, model_cur.factors)]
    candidate = FactorSet(factors, extrap(model_cur.lam, model_prev.lam))
    if error_fn(candidate) < error_fn(model_cur):
        return candidate, True
    return model_cur, False
