"""Per-mode NNLS factor updates on the device (reference: nncp/updaters.py).

In scope (BASELINE north star): MU (updaters.py:91-94), HALS (97-118) and
ANLS-BPP (121-164).  Each call is one fused kernel: optional Hadamard-of-Grams
prologue, the row-parallel update, and fixed-order column reductions.

UCP / ADMM / Nesterov are outside this round's hot-path scope; their names
exist so callers get a clear NotImplementedError instead of an AttributeError.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import torch

from . import _lib
from .tensor_ops import Workspace, as_device

__all__ = ["UpdateInputs", "UpdaterState", "BppCyclingError", "mu_update", "hals_update", "bpp_update",
           "ucp_update", "admm_update", "nesterov_update", "MU_EPSILON", "BPP_BACKUP_TRIES",
           "raise_for_status", "local_reduce"]

MU_EPSILON = 1e-16        # updaters.py:27 (compiled into the kernel)
BPP_BACKUP_TRIES = 3      # updaters.py:28 (compiled into the kernel)


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
    admm_dual: object = None
    nesterov_prev: object = None
    last_inner_iters: int = 0


def raise_for_status(status_host, warn_hals: bool = True):
    """Translate the kernel status words into the reference's warnings / exceptions."""
    mask = (int(status_host[0]) & 0xFFFFFFFF) | ((int(status_host[1]) & 0xFFFFFFFF) << 32)
    if warn_hals and mask:
        for r in range(64):
            if (mask >> r) & 1:
                warnings.warn(f"zero gram diagonal in column {r}, skipping")
    kind = int(status_host[3])
    if kind == 1:
        raise BppCyclingError(int(status_host[2]))
    if kind == 2:
        raise torch.linalg.LinAlgError("Singular matrix")  # numpy.linalg.LinAlgError analogue


def _run(algo: str, inp: UpdateInputs) -> torch.Tensor:
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
    _lib.check(lib.nncp_update(_lib.ALGO_CODES[algo], _lib.ptr(s), 0, -1, r, _lib.ptr(m), _lib.ptr(cur), None,
                               rows, _lib.ptr(out), None, None, _lib.ptr(status), ws.ptr, ws.nbytes, st))
    raise_for_status(status.cpu().tolist(), warn_hals=(algo == "hals"))
    return out


def mu_update(inp: UpdateInputs, eps: float = MU_EPSILON) -> torch.Tensor:
    """H <- H * M / (H S + 1e-16) (updaters.py:91-94)."""
    if eps != MU_EPSILON:
        raise NotImplementedError("the device MU kernel uses the reference epsilon 1e-16")
    return _run("mu", inp)


def hals_update(inp: UpdateInputs, hook=local_reduce) -> torch.Tensor:
    """One Gauss-Seidel column sweep (updaters.py:97-118).

    The reference's per-column hook All-Reduce returns a value nobody reads
    (updaters.py:117); the device path does not issue it.
    """
    return _run("hals", inp)


def bpp_update(inp: UpdateInputs) -> torch.Tensor:
    """Exact NNLS per row by block principal pivoting (updaters.py:121-164)."""
    return _run("bpp", inp)


def _out_of_scope(name):
    def fn(*args, **kwargs):
        raise NotImplementedError(
            f"{name} is outside this build's hot-path scope (MU, HALS, ANLS-BPP); see DESIGN.md")
    fn.__name__ = name
    return fn


ucp_update = _out_of_scope("ucp_update")
admm_update = _out_of_scope("admm_update")
nesterov_update = _out_of_scope("nesterov_update")
