"""Seeded synthetic inputs with the BASELINE.json shapes, generated in HBM.

Stand-in for the reference's `generate_synthetic` (tensor_io.py:103-125), which
caps tensors at 2^27 elements and is noise-free; the BASELINE configs need up
to 8.6e9 elements with |Gaussian| noise.  Truth factors are drawn on the host
with the reference's keying (Philox(key=[seed, (1<<32) | mode]),
tensor_io.py:100,113-120); the tensor itself is produced by the
`nncp_synthetic` kernel (sum of rank-one terms + eta * rms * |N(0,1)| with a
counter-based Philox per global element).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .tensor_ops import DenseTensor, as_device

__all__ = ["truth_factors", "synthetic_block", "synthetic_tensor", "clean_rms"]

_SALT = np.uint64(1) << np.uint64(32)


def truth_factors(dims, rank, seed, kind="uniform"):
    """Host truth factors.  ``kind='uniform'``: U[0,1) (configs 1,2,3,5);
    ``kind='walk'``: temporally smooth nonneg random walks (config 4)."""
    out = []
    for mode, rows in enumerate(dims):
        key = np.array([np.uint64(seed), _SALT | np.uint64(mode)], dtype=np.uint64)
        gen = np.random.Generator(np.random.Philox(key=key))
        if kind == "uniform":
            out.append(gen.random((rows, rank)))
        elif kind == "walk":
            start = gen.random((1, rank))
            steps = gen.standard_normal((rows, rank)) / np.sqrt(rows)
            h = np.maximum(start + np.cumsum(steps, axis=0), 0.0)
            dead = ~(h > 0).any(axis=0)
            if dead.any():
                h[:, dead] = np.abs(gen.standard_normal((rows, int(dead.sum()))))
            out.append(h)
        else:
            raise ValueError(f"unknown factor kind {kind!r}")
    return out


def clean_rms(factors) -> float:
    """rms of sum_r prod_n H_n(i_n, r), from the Gram identity ||X||^2 = 1'(o_n H_n'H_n)1."""
    g = np.ones((factors[0].shape[1],) * 2)
    size = 1
    for h in factors:
        g = g * (h.T @ h)
        size *= h.shape[0]
    return float(np.sqrt(max(g.sum(), 0.0) / size))


def synthetic_block(global_dims, factors, eta, seed, offsets=None, local_dims=None, out=None):
    """Generate one (grid) block of the synthetic tensor on the current GPU."""
    lib = _lib.load()
    gdims = tuple(int(d) for d in global_dims)
    ldims = tuple(int(d) for d in (local_dims or gdims))
    offs = tuple(int(o) for o in (offsets or (0,) * len(gdims)))
    rank = int(factors[0].shape[1])
    noise = float(eta) * clean_rms(factors) if eta else 0.0
    blocks = [as_device(np.ascontiguousarray(h[o:o + l])) for h, o, l in zip(factors, offs, ldims)]
    n = int(np.prod(ldims))
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=blocks[0].device)
    _lib.check(lib.nncp_synthetic(_lib.ptr(out), len(gdims), _lib.i64(ldims), _lib.i64(offs), _lib.i64(gdims),
                                  _lib.ptrs(blocks), rank, noise, int(seed) & (2**64 - 1), _lib.stream_handle()))
    torch.cuda.current_stream().synchronize()
    return out


def synthetic_tensor(dims, rank, seed=1, eta=0.01, kind="uniform") -> DenseTensor:
    """Device-resident DenseTensor for one BASELINE config."""
    fs = truth_factors(dims, rank, seed, kind)
    return DenseTensor(dims, synthetic_block(dims, fs, eta, seed))
