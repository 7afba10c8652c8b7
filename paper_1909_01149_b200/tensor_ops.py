"""Dense tensor / factor containers and the small device primitives.

Mirrors the reference module `nncp/tensor_ops.py` (layout contract at
tensor_ops.py:1-13): a tensor is a flat float64 buffer with the mode-1 index
fastest; factors are row-major (I_n, R).  Containers accept host numpy arrays
or torch tensors; every numeric routine here runs on the GPU through
libnncp_b200.so (no CPU fallback).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "DenseTensor", "FactorSet", "gram", "hadamard_grams_excluding", "khatri_rao", "matrix_inner_product",
    "naive_mttkrp", "norm_squared", "normalize_columns", "reconstruct", "device", "as_device", "Workspace",
]


def on_host(*objs) -> bool:
    """True unless one of ``objs`` (arrays, tensors, DenseTensors, lists of them) lives
    on the GPU: the operator-level functions answer host inputs with numpy arrays,
    like the reference, and device inputs with device tensors."""
    for o in objs:
        if isinstance(o, (list, tuple)):
            if not on_host(*o):
                return False
        elif isinstance(o, torch.Tensor) and o.is_cuda:
            return False
        elif isinstance(o, DenseTensor) and o.on_device:
            return False
        elif isinstance(o, FactorSet) and not on_host(*o.factors):
            return False
    return True


def to_host_if(t, host: bool):
    """``t`` as a numpy array when the call's inputs were host arrays."""
    return t.detach().cpu().numpy() if host and isinstance(t, torch.Tensor) else t


def device() -> torch.device:
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def as_device(a, dtype=torch.float64) -> torch.Tensor:
    """Contiguous float64 CUDA tensor view/copy of ``a`` (numpy or torch)."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    if t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.to(device(), non_blocking=False)
    return t.contiguous()


class Workspace:
    """Zero-filled device scratch shared by the kernels of one execution context."""

    def __init__(self, nbytes: int):
        n = (int(nbytes) + 7) // 8 + 64
        self.buf = torch.zeros(n, dtype=torch.float64, device=device())
        self.nbytes = self.buf.numel() * 8

    def grow(self, nbytes: int):
        if nbytes > self.nbytes:
            torch.cuda.current_stream().synchronize()
            self.__init__(nbytes)

    @property
    def ptr(self):
        return _lib.vp(self.buf.data_ptr())


_default_ws = {}


def default_workspace(nbytes: int = 1 << 20) -> Workspace:
    dev = torch.cuda.current_device()
    ws = _default_ws.get(dev)
    if ws is None:
        ws = _default_ws[dev] = Workspace(max(nbytes, 1 << 20))
    ws.grow(nbytes)
    return ws


class DenseTensor:
    """Dense N-way tensor over a flat mode-1-fastest float64 buffer (tensor_ops.py:23-78).

    ``data`` may be a numpy array (host) or a torch tensor (host or CUDA).
    """

    __slots__ = ("dims", "data")

    def __init__(self, dims, data=None):
        dims = tuple(int(d) for d in dims)
        if len(dims) < 2:
            raise ValueError("tensor order must be at least 2")
        if any(d < 1 for d in dims):
            raise ValueError(f"dims must be positive, got {dims}")
        size = int(np.prod(dims))
        if data is None:
            data = np.zeros(size)
        elif isinstance(data, torch.Tensor):
            data = data.reshape(-1)
            if data.dtype != torch.float64:
                data = data.to(torch.float64)
            data = data.contiguous()
            if data.numel() != size:
                raise ValueError(f"data length {data.numel()} does not match prod(dims) {size}")
        else:
            data = np.ascontiguousarray(data, dtype=np.float64).ravel()
            if data.size != size:
                raise ValueError(f"data length {data.size} does not match prod(dims) {size}")
        self.dims = dims
        self.data = data

    @classmethod
    def from_array(cls, arr):
        arr = np.asarray(arr, dtype=np.float64)
        return cls(arr.shape, arr.ravel(order="F"))

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def size(self) -> int:
        return int(np.prod(self.dims))

    @property
    def on_device(self) -> bool:
        return isinstance(self.data, torch.Tensor) and self.data.is_cuda

    def to_device(self) -> "DenseTensor":
        """Same tensor with its buffer resident in HBM.

        From page-locked host memory the copy is queued asynchronously on the
        current stream, so the engine's allocations (the sliced tensor, tens of GB
        at the BASELINE sizes) and host-side setup overlap the transfer; every
        consumer is ordered behind it on the stream.
        """
        if self.on_device:
            return self
        d = self.data
        if isinstance(d, torch.Tensor) and d.is_pinned() and d.dtype == torch.float64 and d.is_contiguous():
            out = torch.empty(d.numel(), dtype=torch.float64, device=device())
            out.copy_(d.reshape(-1), non_blocking=True)
            return DenseTensor(self.dims, out)
        return DenseTensor(self.dims, as_device(d))

    def host_data(self) -> np.ndarray:
        if isinstance(self.data, torch.Tensor):
            return self.data.detach().cpu().numpy()
        return self.data

    def as_array(self):
        """Host N-d view indexed as a[i_1, ..., i_N]."""
        return self.host_data().reshape(self.dims, order="F")

    def unfold_leading(self, split: int):
        if not 1 <= split < self.order:
            raise ValueError(f"split must be in [1, {self.order - 1}], got {split}")
        rows = int(np.prod(self.dims[:split]))
        return self.host_data().reshape((rows, -1), order="F")

    def norm_squared(self) -> float:
        return norm_squared(self)


@dataclass
class FactorSet:
    """N factor matrices sharing rank R plus column weights (tensor_ops.py:81-118)."""

    factors: list
    lam: object = None

    def __post_init__(self):
        self.factors = [f if isinstance(f, torch.Tensor) else np.asarray(f, dtype=np.float64)
                        for f in self.factors]
        ranks = {int(h.shape[1]) for h in self.factors}
        if len(ranks) != 1:
            raise ValueError(f"factors disagree on rank: {sorted(ranks)}")
        if self.lam is None:
            self.lam = np.ones(self.rank)
        elif not isinstance(self.lam, torch.Tensor):
            self.lam = np.asarray(self.lam, dtype=np.float64)
            if self.lam.shape != (self.rank,):
                raise ValueError("lambda length must equal the rank")

    @property
    def order(self) -> int:
        return len(self.factors)

    @property
    def rank(self) -> int:
        return int(self.factors[0].shape[1])

    @property
    def dims(self):
        return tuple(int(h.shape[0]) for h in self.factors)

    def copy(self) -> "FactorSet":
        cp = lambda a: a.clone() if isinstance(a, torch.Tensor) else a.copy()  # noqa: E731
        return FactorSet([cp(h) for h in self.factors], cp(self.lam))

    def to_host(self) -> "FactorSet":
        h = lambda a: a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a  # noqa: E731
        return FactorSet([h(f) for f in self.factors], h(self.lam))


# ------------------------------------------------------------ device ops ----

def norm_squared(x: DenseTensor) -> float:
    """||X||^2 on the device (tensor_ops.py:76-78)."""
    lib = _lib.load()
    d = x.to_device().data
    out = torch.empty(1, dtype=torch.float64, device=d.device)
    ws = default_workspace(1 << 20)
    _lib.check(lib.nncp_norm_squared(_lib.ptr(d), d.numel(), _lib.ptr(out), ws.ptr, ws.nbytes,
                                     _lib.stream_handle()))
    return float(out.item())


def gram(h):
    """H^T H forced symmetric (tensor_ops.py:140-143); device kernel + 0.5(G+G^T)."""
    if on_host(h):
        return to_host_if(gram(as_device(h)), True)
    lib = _lib.load()
    h = as_device(h)
    rows, r = int(h.shape[0]), int(h.shape[1])
    g = torch.empty((r, r), dtype=torch.float64, device=h.device)
    ws = default_workspace(256 + 8 * (r * r * max(1, (rows + 63) // 64) + 1024))
    _lib.check(lib.nncp_gram(_lib.ptr(h), rows, r, _lib.ptr(g), ws.ptr, ws.nbytes, _lib.stream_handle()))
    return 0.5 * (g + g.T)


def hadamard_grams_excluding(grams, exclude: int):
    """Elementwise product of all Grams except ``exclude`` (tensor_ops.py:146-155)."""
    if not 0 <= exclude < len(grams):
        raise ValueError(f"exclude index {exclude} out of range")
    if on_host(list(grams)):
        return to_host_if(hadamard_grams_excluding([as_device(g) for g in grams], exclude), True)
    out = None
    for m, g in enumerate(grams):
        if m != exclude:
            g = as_device(g)
            out = g.clone() if out is None else out * g
    if out is None:
        r = int(as_device(grams[0]).shape[0])
        out = torch.ones((r, r), dtype=torch.float64, device=device())
    return out


def matrix_inner_product(a, b) -> float:
    """Frobenius inner product on the device (tensor_ops.py:208-212)."""
    lib = _lib.load()
    a, b = as_device(a), as_device(b)
    if tuple(a.shape) != tuple(b.shape):
        raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    rows = int(a.shape[0]) if a.dim() > 1 else 1
    r = int(a.numel() // max(rows, 1)) if a.numel() else 1
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    ws = default_workspace(1 << 20)
    _lib.check(lib.nncp_inner(_lib.ptr(a), _lib.ptr(b), None, rows, r, _lib.ptr(out), ws.ptr, ws.nbytes,
                              _lib.stream_handle()))
    return float(out.item())


def normalize_columns(h):
    """Unit columns and their norms (tensor_ops.py:198-205), via the fused device kernel."""
    if on_host(h):
        out, lam = normalize_columns(as_device(h))
        return to_host_if(out, True), to_host_if(lam, True)
    lib = _lib.load()
    h = as_device(h)
    rows, r = int(h.shape[0]), int(h.shape[1])
    ws = default_workspace(256 + 8 * (r * r * max(1, (rows + 63) // 64) + 1024))
    nsq = torch.empty(r, dtype=torch.float64, device=h.device)
    # column sums of squares = the raw Gram diagonal (fixed-order device reduction)
    g = torch.empty((r, r), dtype=torch.float64, device=h.device)
    _lib.check(lib.nncp_gram(_lib.ptr(h), rows, r, _lib.ptr(g), ws.ptr, ws.nbytes, _lib.stream_handle()))
    nsq.copy_(torch.diagonal(g))
    out = torch.empty_like(h)
    lam = torch.empty(r, dtype=torch.float64, device=h.device)
    _lib.check(lib.nncp_normalize_gram(_lib.ptr(h), _lib.ptr(nsq), rows, r, _lib.ptr(out), _lib.ptr(lam),
                                       _lib.ptr(g), ws.ptr, ws.nbytes, _lib.stream_handle()))
    return out, lam


def khatri_rao(factors):
    """Khatri-Rao product, first factor's index fastest (tensor_ops.py:121-137), built by
    the device kernel nncp_khatri_rao (the hot path never materialises it)."""
    factors = list(factors)
    if len(factors) == 0:
        raise ValueError("khatri_rao needs at least one factor")
    ranks = {int(h.shape[1]) for h in factors}
    if len(ranks) != 1:
        raise ValueError(f"khatri_rao rank mismatch: {sorted(ranks)}")
    host = on_host(factors)
    r = ranks.pop()
    if len(factors) > _lib.MAX_ORDER:          # fold the tail first: same rows, same order
        factors = factors[:_lib.MAX_ORDER - 1] + [khatri_rao(factors[_lib.MAX_ORDER - 1:])]
    dev = [as_device(h) for h in factors]
    rows = [int(h.shape[0]) for h in dev]
    out = torch.empty((int(np.prod(rows)), r), dtype=torch.float64, device=dev[0].device)
    lib = _lib.load()
    _lib.check(lib.nncp_khatri_rao(_lib.ptrs(dev), _lib.i64(rows), len(dev), r, _lib.ptr(out),
                                   _lib.stream_handle()))
    return to_host_if(out, host)


def naive_mttkrp(x: DenseTensor, factors, mode: int):
    """MTTKRP in ``mode`` (tensor_ops.py:158-185), the reference's oracle path.

    The reference sums with one einsum over the dense array; here the same quantity
    comes from the device kernels without a dimension tree: one partial MTTKRP on the
    side of the root split that retains ``mode`` and a multi-TTV chain
    (DimTreeContext.mttkrp_direct)."""
    from .dimtree import DimTreeContext, DimTreePlan

    hs = list(factors.factors) if isinstance(factors, FactorSet) else list(factors)
    n = x.order
    if len(hs) != n:
        raise ValueError("factor count does not match tensor order")
    for m, h in enumerate(hs):
        if m != mode and int(h.shape[0]) != x.dims[m]:
            raise ValueError(f"factor {m} has {int(h.shape[0])} rows, tensor dim is {x.dims[m]}")
    if n > _lib.MAX_ORDER:
        raise ValueError("tensor order too large for naive path")
    if not 0 <= mode < n:
        raise ValueError(f"mode {mode} out of range")
    host = on_host(x, hs)
    ranks = {int(h.shape[1]) for h in hs}
    if len(ranks) != 1:
        raise ValueError(f"factors disagree on rank: {sorted(ranks)}")
    plan = DimTreePlan.create(x.dims, ranks.pop())
    out = DimTreeContext(plan).mttkrp_direct(x, hs, mode)
    return to_host_if(out, host)


def reconstruct(model: FactorSet) -> DenseTensor:
    """Dense tensor of the model, sum_r lam_r prod_n H_n(i_n, r) (tensor_ops.py:192-195),
    generated by the device kernel (nncp_synthetic with no noise)."""
    from .synth import synthetic_block

    host = on_host(model)
    fs = [f.detach().cpu().numpy() if isinstance(f, torch.Tensor) else np.asarray(f, dtype=np.float64)
          for f in model.factors]
    lam = model.lam.detach().cpu().numpy() if isinstance(model.lam, torch.Tensor) else np.asarray(model.lam)
    fs[0] = fs[0] * lam[None, :]
    data = synthetic_block(model.dims, fs, 0.0, 0)
    return DenseTensor(model.dims, to_host_if(data, host))
