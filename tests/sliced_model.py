"""Bit-exact numpy model of the sliced-tensor partial MTTKRP.

TEST INFRASTRUCTURE ONLY.  It restates, operation by operation, what
paper_1909_01149_b200/csrc/mttkrp_sliced.cu computes -- the row exponents and
balanced base-256 digits of X_(1:S), the per-(chunk, column) exponents and
digits of the Khatri-Rao side, the exact integer level sums of the tensor-core
MMAs, the fp64 epilogue (levels grouped in exact int64, power-of-two scaling,
chunk-ordered accumulation) and the split-K group plan and fixed-order group
reduction -- so that

* on a GPU, the kernel's output must equal ``sliced_partial`` bit for bit (the
  kernel does exactly the designed integer algorithm: no dropped MMAs, no
  races), and
* on a CPU, ``sliced_partial`` against the oracle (oracle/nncp_oracle.py, the
  reference restatement) checks the error model itself.
"""

from __future__ import annotations

import math

import numpy as np

BM = 128
BK = 128
KC_MAX = 16384
SEG_G = 16


def _align(v, a):
    return -(-v // a) * a


def _frexp_exp(v):
    """frexp exponents (0 for zeros), elementwise."""
    _, e = np.frexp(v)
    return np.where(v == 0, 0, e).astype(np.int64)


def _digits(scaled, levels):
    """Balanced base-256 digits of rint(scaled) (round half to even): list of int64 arrays, d_0 first."""
    q = np.rint(scaled).astype(np.int64)
    c = (1 << (8 * (levels - 1))) // 255 * 128
    u = q + c
    out = [u >> (8 * (levels - 1))]
    for s in range(1, levels):
        out.append(((u >> (8 * (levels - 1 - s))) & 255) - 128)
    return out


def plan(dims, split, side, rank, sms=148):
    """Mirror of sliced::plan_call (chunk length, chunk count, split-K groups)."""
    m = math.prod(dims[:split])
    j = math.prod(dims[split:])
    mp, jp = _align(m, BM), _align(j, BK)
    left = side == "left"
    k, kp = (j, jp) if left else (m, mp)
    rows = m if left else j
    row_tiles = (mp if left else jp) // BM
    if left and row_tiles >= sms:
        groups = 1
        kc = min(KC_MAX, _align(kp, 256))
    else:
        want = max(1, sms // row_tiles)
        per_group = -(-kp // want)
        q = max(1, -(-per_group // KC_MAX))
        kc = min(KC_MAX, max(256, _align(-(-kp // (want * q)), 256)))
        nch = -(-kp // kc)
        groups = min(want, nch)
    nchunks = -(-kp // kc)
    return dict(M=m, J=j, K=k, Kp=kp, rows=rows, Kc=kc, nchunks=nchunks, groups=groups,
                RP=_align(rank, 16))


def _krp_values(factors, dims_used, rank, order_seg):
    """KRP rows (first factor fastest) with the kernel's multiplication order:
    left to right, or h0 * (h1 * h2 ...) on the segment-reuse path."""
    n = len(factors)
    k = math.prod(dims_used)
    idx = np.arange(k, dtype=np.int64)
    digs = []
    for d in dims_used:
        digs.append(idx % d)
        idx = idx // d
    if order_seg:
        g = np.ones((k, rank))
        for f in range(1, n):
            g = g * factors[f][digs[f]]
        return factors[0][digs[0]] * g
    v = factors[0][digs[0]].copy()
    for f in range(1, n):
        v = v * factors[f][digs[f]]
    return v


def sliced_partial(x, dims, split, side, factors, rank, levels=6, sms=148):
    """Sliced partial MTTKRP exactly as the kernel computes it; returns the flat
    column-major (retained, R) output (TempTensor layout)."""
    dims = tuple(int(d) for d in dims)
    x = np.asarray(x, dtype=np.float64).ravel()
    p = plan(dims, split, side, rank, sms)
    m, j = p["M"], p["J"]
    xm = x.reshape(j, m).T                               # X_(1:S): (M, J) column-major view
    # ---- slice X once: row exponents and digits
    rowmax = np.abs(xm).max(axis=1)
    ex = _frexp_exp(rowmax)
    xd = _digits(np.ldexp(xm, (8 * levels - 2 - ex)[:, None]), levels)
    # ---- factor side
    if side == "left":
        used = list(range(split, len(dims)))
    else:
        used = list(range(split))
    fs = [np.asarray(factors[u], dtype=np.float64) for u in used]
    dused = [dims[u] for u in used]
    nf = len(fs)
    seg = nf >= 2 and nf <= 3 and dused[0] % BK == 0
    b = _krp_values(fs, dused, rank, seg)                  # (K, R)
    if side == "right":
        b = np.ldexp(b, ex[:, None])                     # fold 2^rowexp[m] into B
    k = p["K"]
    kc, nch = p["Kc"], p["nchunks"]
    chunk_of = np.arange(k) // kc
    eb = np.zeros((nch, rank), dtype=np.int64)
    none = np.ones((nch, rank), dtype=bool)
    for c in range(nch):
        sl = slice(c * kc, min(k, (c + 1) * kc))
        mx = np.abs(b[sl]).max(axis=0) if sl.start < k else np.zeros(rank)
        none[c] = mx == 0
        eb[c] = np.where(mx == 0, 0, _frexp_exp(mx))
    kx = 8 * levels - 2 - eb[chunk_of]                   # (K, R)
    bd = _digits(np.ldexp(b, kx), levels)
    # ---- integer GEMM per chunk + fp64 epilogue
    if side == "left":
        a_d = xd                                         # rows m, contraction j
        rows = m
        row_e = ex
    else:
        a_d = [d.T for d in xd]                          # rows j, contraction m
        rows = j
        row_e = np.zeros(j, dtype=np.int64)
    groups = p["groups"]
    parts = []
    for g in range(groups):
        c0, c1 = g * nch // groups, (g + 1) * nch // groups
        acc = np.zeros((rows, rank))
        for c in range(c0, c1):
            sl = slice(c * kc, min(k, (c + 1) * kc))
            if sl.start >= k:
                continue
            lev = []
            for lvl in range(levels):
                t = np.zeros((rows, rank), dtype=np.int64)
                for s in range(lvl + 1):
                    t += a_d[s][:, sl] @ bd[lvl - s][sl]
                lev.append(t)
            # the kernel's epilogue: levels combined three at a time in exact int64,
            # one fp64 rounding per pair of groups (L = 7: the seventh level joins
            # the low group first)
            g1 = lev[0] * 65536 + lev[1] * 256 + lev[2]
            g2 = lev[3] * 65536 + lev[4] * 256 + lev[5]
            low = g2.astype(np.float64)
            if levels == 7:
                low = low + lev[6].astype(np.float64) * 2.0 ** -8
            v = (g1.astype(np.float64) + low * 2.0 ** -24) * 2.0 ** -16
            e = row_e[:, None] + np.where(none[c], 0, eb[c])[None, :] - 12
            acc = acc + np.ldexp(v, e)
        parts.append(acc)
    out = parts[0]
    for g in range(1, groups):
        out = out + parts[g]
    return out.T.ravel()                                 # [r][row]
