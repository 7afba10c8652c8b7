"""NNCP alternating-update driver on B200 (reference: nncp/driver.py).

Public surface identical to the reference (driver.py:46-56, 73-134, 495-531):
``RunConfig``, ``RunReport``, ``record_category``, ``init_factor``,
``relative_error``, ``nncp_sequential``, ``nncp_parallel``, ``CATEGORIES``,
``ALGORITHMS``.  The inner program is the reference's ``_run_spmd``
(driver.py:331-449) with every numeric step on the GPU:

    per mode n:  MTTKRP (dimension tree: DMMA partial GEMMs + TTV kernels)
                 -> Reduce-Scatter(slice)            [identity on one GPU]
                 -> fused Hadamard + MU/HALS/BPP update + column sums (+ beta)
                 -> All-Reduce(nsq) -> fused normalise + Gram -> All-Reduce(Gram)
                 -> All-Gather(slice)
    per sweep:   All-Reduce(beta), gamma kernel, one 2-scalar + status D2H

Host work per iteration is kernel launches plus that one small read-back;
by default the whole sweep is replayed as a CUDA graph after the first one
(``RunConfig.cuda_graph``).
Category seconds come from CUDA events on the launching stream.
"""

from __future__ import annotations

import math
import os
import threading
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .dimtree import DeferredPartial, DimTreeContext, DimTreePlan, SlicedTensor, choose_balanced_split
from .grid import (CommCounters, DistCollectives, Grid, IdentityCollectives, RankLayout, ThreadCollectives,
                   ThreadGrid, block_partition)
from .tensor_ops import DenseTensor, FactorSet, Workspace, as_device
from .updaters import (AdmmRunner, BppCyclingError, NesterovRunner, _SPack,  # noqa: F401
                       raise_for_code, raise_for_status, warn_for_status)

__all__ = ["ALGORITHMS", "CATEGORIES", "RunConfig", "RunReport", "init_factor", "nncp_parallel",
           "nncp_sequential", "record_category", "relative_error", "IN_SCOPE_ALGORITHMS", "run_local"]

CATEGORIES = ("MTTKRP", "KRP", "MultiTTV", "Gram", "NNLS", "ReduceScatter", "AllGather", "AllReduce", "Error")
ALGORITHMS = ("ucp", "mu", "hals", "bpp", "admm", "nes")
IN_SCOPE_ALGORITHMS = ALGORITHMS          # all six update rules run on the device
FUSED_ALGORITHMS = ("mu", "hals", "bpp", "ucp")   # one kernel per mode (CUDA-graph capturable)


@dataclass
class RunConfig:
    """Knobs of one decomposition run (driver.py:73-101).

    ``cuda_graph`` (device-only): after the first sweep, the whole sweep of
    launches (including the per-category timing events) is replayed as one
    CUDA graph.  ``None`` (default) enables it whenever the sweep is
    capturable (MU/HALS/BPP/UCP, one execution context or one process per GPU
    with in-place NCCL collectives, which are captured with the kernels);
    ``False`` forces eager launches.
    """

    rank: int
    algorithm: str = "bpp"
    max_iters: int = 100
    tol: float = 1e-6
    seed: int = 0
    grid: tuple = None
    use_dimtree: bool = True
    strict_split: bool = False
    initial_factors: FactorSet = None
    cuda_graph: bool = None   # None = auto: replay the sweep as a CUDA graph when it is capturable
    # partial-MTTKRP engine: "sliced" = int8 tensor cores over a once-sliced tensor
    # (DESIGN.md §4.4), "fp64" = FP64 DMMA, "auto" = sliced when its cost model wins
    # and the slices fit in HBM
    mttkrp_kernel: str = "auto"
    # digit levels of the sliced engine: 6 (46-bit operands, 6 B/element) or 7 (54-bit,
    # for rows spanning extreme dynamic ranges; 7 B/element)
    mttkrp_levels: int = 6
    # dimension-tree root split: "reference" = the reference rule (first S with
    # M >= J, dimtree.py:25-39); "auto" = that rule, except that the sliced engine
    # takes the split minimising M + J when it at least halves it
    dimtree_split: str = "auto"
    # ANLS-BPP: start each row's block principal pivoting from the passive set it ended
    # with in the previous outer iteration instead of P = {} (updaters.py:121-155).  The
    # minimiser is unique for SPD S and the final pass solves on the final passive set,
    # so the result is the reference's; False = the reference's cold start every time.
    bpp_warm_start: bool = True

    def validate(self, order: int):
        if self.rank < 1:
            raise ValueError("rank must be at least 1")
        if self.tol < 0:
            raise ValueError("tolerance must be nonnegative")
        if self.max_iters < 0:
            raise ValueError("max_iters must be nonnegative")
        if self.algorithm not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if self.grid is not None and len(self.grid) != order:
            raise ValueError(f"grid order {len(self.grid)} does not match tensor order {order}")
        if self.initial_factors is not None and self.initial_factors.rank != self.rank:
            raise ValueError("initial factors disagree with configured rank")
        if self.algorithm not in IN_SCOPE_ALGORITHMS:
            raise NotImplementedError(
                f"algorithm {self.algorithm!r} is outside this build's hot-path scope "
                f"(supported: {', '.join(IN_SCOPE_ALGORITHMS)})")
        if self.mttkrp_kernel not in ("auto", "sliced", "fp64"):
            raise ValueError(f"unknown mttkrp_kernel {self.mttkrp_kernel!r} (auto, sliced, fp64)")
        if self.dimtree_split not in ("auto", "reference"):
            raise ValueError(f"unknown dimtree_split {self.dimtree_split!r} (auto, reference)")
        if self.mttkrp_levels not in (6, 7):
            raise ValueError(f"mttkrp_levels must be 6 or 7, got {self.mttkrp_levels!r}")
        if self.rank > _lib.MAX_RANK:
            raise NotImplementedError(f"rank {self.rank} exceeds the device limit {_lib.MAX_RANK}")
        if order > _lib.MAX_ORDER:
            raise NotImplementedError(f"tensor order {order} exceeds the device limit {_lib.MAX_ORDER}")


@dataclass
class RunReport:
    """Error curve plus timing / communication breakdown (driver.py:104-126)."""

    errors: list = field(default_factory=list)
    rows: list = field(default_factory=list)
    row_words: list = field(default_factory=list)
    row_wall: list = field(default_factory=list)
    counters: CommCounters = field(default_factory=CommCounters)
    model: FactorSet = None
    converged: bool = False
    split_mode: int = None
    tree_partial_calls: int = 0

    def begin_row(self):
        self.rows.append({c: 0.0 for c in CATEGORIES})
        self.row_words.append(0)
        self.row_wall.append(0.0)


def record_category(report: RunReport, category: str, elapsed: float, words: int = 0):
    """driver.py:129-134."""
    if category not in CATEGORIES:
        raise ValueError(f"unknown category {category!r}")
    report.rows[-1][category] += elapsed
    report.row_words[-1] += words


def init_factor(seed: int, mode: int, rows: int, rank: int) -> np.ndarray:
    """Uniform [0,1) factor, Philox keyed by (seed, mode) (driver.py:137-143).

    Generated on the host with numpy's Philox so the draws are bit-identical
    to the reference; uploaded once per run.
    """
    key = np.array([np.uint64(seed), np.uint64(mode)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key)).random((rows, rank))


def _eps_from_terms(alpha: float, beta: float, gamma: float) -> float:
    """driver.py:146-148 (host arithmetic on three device-reduced scalars)."""
    return float(np.sqrt(max(0.0, alpha - 2.0 * beta + gamma) / alpha))


def relative_error(alpha, mttkrp_n, h_n_unnormalized, s_n, g_n, lam) -> float:
    """driver.py:151-162 with beta / gamma reduced on the device."""
    if alpha <= 0.0:
        raise ValueError("zero tensor has no relative error")
    lib = _lib.load()
    m = as_device(mttkrp_n)
    h = as_device(h_n_unnormalized)
    if tuple(m.shape) != tuple(h.shape):
        raise ValueError(f"shape mismatch: {tuple(m.shape)} vs {tuple(h.shape)}")
    r = int(m.shape[1])
    lam_d = as_device(lam)
    pair = torch.stack([as_device(s_n), as_device(g_n)]).contiguous()
    out = torch.empty(2, dtype=torch.float64, device=m.device)
    ws = Workspace(1 << 20)
    st = _lib.stream_handle()
    _lib.check(lib.nncp_inner(_lib.ptr(m), _lib.ptr(h), None, int(m.shape[0]), r, _lib.ptr(out), ws.ptr, ws.nbytes,
                              st))
    _lib.check(lib.nncp_gamma(_lib.ptr(pair), 2, r, _lib.ptr(lam_d), _lib.vp(out.data_ptr() + 8), st))
    beta, gamma = out.cpu().tolist()
    return _eps_from_terms(float(alpha), beta, gamma)


# ------------------------------------------------------------ timing --------

class _EventTimer:
    """Category seconds from CUDA events recorded at phase boundaries."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self._pool = []
        self._marks = []
        self._start = None
        self.capturing = False          # marks become event-record nodes of the sweep graph
        self.graph_marks = None         # (start, [(category, tag, event), ...]) of the captured sweep
        # tag -> [seconds, count]: finer intervals inside a category (e.g. each partial
        # MTTKRP launch, "partial_left" / "partial_right"), accumulated like the rows
        self.tags = {}

    def _event(self):
        if self.capturing:
            return torch.cuda.Event(enable_timing=True, external=True)
        if self._pool:
            return self._pool.pop()
        return torch.cuda.Event(enable_timing=True)

    def begin_capture(self):
        self.capturing = True
        self.start()

    def end_capture(self):
        if self.enabled:
            self.graph_marks = (self._start, list(self._marks))
        self._marks, self._start = [], None
        self.capturing = False

    def collect_marks(self, graph_marks, row: dict):
        """Per-category seconds of a finished graph replay whose marks are ``graph_marks``."""
        if not self.enabled or graph_marks is None:
            return
        prev, marks = graph_marks
        for cat, tag, e in marks:
            dt = prev.elapsed_time(e) / 1e3
            row[cat] += dt
            self._tag(tag, dt)
            prev = e

    def _tag(self, tag, dt):
        if tag is not None:
            acc = self.tags.setdefault(tag, [0.0, 0])
            acc[0] += dt
            acc[1] += 1

    def start(self):
        if not self.enabled:
            return
        self._start = self._event()
        self._start.record()
        self._marks = []

    def mark(self, category, tag=None):
        """Close the interval since the previous mark and attribute it to ``category``
        (and, when given, to ``tag``)."""
        if not self.enabled:
            return
        e = self._event()
        e.record()
        self._marks.append((category, tag, e))

    def collect(self, row: dict):
        """Accumulate (after the stream is synchronised) into ``row``."""
        if not self.enabled or self._start is None:
            return
        prev = self._start
        for cat, tag, e in self._marks:
            dt = prev.elapsed_time(e) / 1e3
            row[cat] += dt
            self._tag(tag, dt)
            self._pool.append(prev)
            prev = e
        self._pool.append(prev)
        self._marks = []
        self._start = None


# ------------------------------------------------------------ engine --------

SLICED_MIN_ELEMS = 1 << 22       # below this the fp64 path's fewer launches win
# rows * R^2 up to which the update kernel's last CTA also normalises and forms the Gram
# (nncp_update_normalize).  Measured: 64^3 R=10 (6.4e3) 0.0904 -> 0.0887 ms/iter; at
# 512^3 R=16 (1.3e5) one CTA doing the Gram is already slower than the separate
# normalise launch (0.412 -> 0.466 ms/iter), at 1024^3 R=32 (1.0e6) far slower.
FUSED_TAIL_MAX = 1 << 14
SLICED_HBM_MARGIN = 4 << 30      # bytes left free after the slices
# partial-MTTKRP cost model for mttkrp_kernel="auto" (B200 measurements):
# FP64 DMMA path reaches ~87% of max(8 I / BW, 2 I R / 37.1 TF); the sliced path streams
# 6 I bytes at ~6.9 TB/s plus ~50 us of per-call digit prep, launches and tail
# (512^3 R=16: 0.155 / 0.176 ms sliced vs 0.196 / 0.185 ms DMMA)
_HBM_BPS, _DMMA_FLOPS, _SLICED_BPS, _SLICED_FIXED_S = 6.45e12, 37.1e12, 6.9e12, 5e-5


# "auto" slices only tensors whose nonzero magnitudes span at most this ratio: the digit
# planes keep 46 bits relative to each row's maximum, so an entry 2^k below it keeps
# 46 - k bits ("Engine choice")
SLICED_MAX_RANGE = 2.0 ** 10


class TensorFacts:
    """What the initial norm pass learns about the local tensor (one read, nncp_norm_squared_min)."""

    __slots__ = ("alpha", "min", "absmax", "absmin_nz")

    def __init__(self, alpha, xmin, absmax, absmin_nz):
        self.alpha, self.min, self.absmax, self.absmin_nz = float(alpha), float(xmin), float(absmax), float(absmin_nz)

    @property
    def finite(self) -> bool:
        return math.isfinite(self.alpha) and math.isfinite(self.absmax)

    @property
    def signed(self) -> bool:
        return self.min < 0.0

    @property
    def dynamic_range(self) -> float:
        if self.absmax == 0.0 or not math.isfinite(self.absmin_nz):
            return 1.0
        return self.absmax / self.absmin_nz


def _sliced_ok_for(facts: TensorFacts, algorithm: str):
    """Why "auto" must not slice this tensor (None = it may).  The Ozaki-scheme bound of
    the sliced engine is relative to row / column-chunk maxima, not to each output: with
    cancellation (signed tensors, or UCP's signed factors) or entries far below their
    row's maximum the relative error of an output can exceed the 1e-12 MTTKRP tolerance
    (tests/test_gpu_sliced.py::test_auto_engine_guards); non-finite entries have no digits."""
    if facts is None:
        return None
    if not facts.finite:
        return "non-finite entries"
    if facts.signed:
        return "negative entries"
    if algorithm == "ucp":
        return "signed (unconstrained) factors"
    if facts.dynamic_range > SLICED_MAX_RANGE:
        return f"nonzero magnitudes span {facts.dynamic_range:.3g}x"
    return None


def _use_sliced(kind: str, dims, split: int, rank: int, dev, levels: int = 6, extra_bytes: int = 0,
                facts: TensorFacts = None, algorithm: str = "hals") -> bool:
    """Resolve RunConfig.mttkrp_kernel for one execution context."""
    if kind == "fp64":
        return False
    if facts is not None and not facts.finite:
        if kind == "sliced":
            warnings.warn("tensor has non-finite entries; the sliced MTTKRP engine cannot represent them, "
                          "using the fp64 engine")
        return False
    if kind == "sliced":
        return True
    if _sliced_ok_for(facts, algorithm) is not None:
        return False
    size = int(np.prod(dims))
    if size < SLICED_MIN_ELEMS:
        return False
    t_fp64 = max(8.0 * size / _HBM_BPS, 2.0 * size * rank / _DMMA_FLOPS) / 0.87
    t_sliced = float(levels) * size / _SLICED_BPS + _SLICED_FIXED_S
    if t_sliced >= t_fp64:
        return False
    free, _ = torch.cuda.mem_get_info(dev)
    free += torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)   # torch's cached blocks
    return SlicedTensor.nbytes(dims, split, levels) + SLICED_HBM_MARGIN + extra_bytes <= free


def _engine_plan(dims, cfg: RunConfig, dev, extra_bytes: int = 0, facts: TensorFacts = None):
    """Dimension-tree plan and partial-MTTKRP engine of one execution context:
    (plan, sliced?).  ``extra_bytes``: device memory still to be allocated first;
    ``facts``: sign / range of the tensor (None before it is on the device)."""
    plan = DimTreePlan.create(dims, int(cfg.rank), cfg.strict_split)
    if not _use_sliced(cfg.mttkrp_kernel, dims, plan.split, int(cfg.rank), dev, cfg.mttkrp_levels, extra_bytes,
                       facts, cfg.algorithm):
        return plan, False
    if cfg.dimtree_split == "auto":
        s_bal = choose_balanced_split(dims)
        if 2 * _split_rows(dims, s_bal) <= _split_rows(dims, plan.split):
            plan = DimTreePlan(dims, int(cfg.rank), s_bal)
    return plan, True


def _reserve_sliced(dims, cfg: RunConfig):
    """Before a host tensor is copied in: allocate and release the sliced tensor's
    buffer through torch's caching allocator while the device is idle.  cudaMalloc
    waits for pending device work, so allocating the ~50 GB buffer behind the
    asynchronous H2D would serialise on the copy; the cached block is reused by
    SlicedTensor with no driver call."""
    dev = torch.device("cuda", torch.cuda.current_device())
    plan, sliced = _engine_plan(dims, cfg, dev, extra_bytes=8 * math.prod(dims))
    if sliced:
        torch.empty(SlicedTensor.nbytes(dims, plan.split, cfg.mttkrp_levels), dtype=torch.uint8, device=dev)


def _split_rows(dims, s: int) -> int:
    """M + J of the root split S: the rows of the two partial outputs and of the Khatri-Rao digit sides."""
    return math.prod(dims[:s]) + math.prod(dims[s:])


def first_failure(vec, nranks: int, order: int):
    """(mode, kind, row) of the first failed update in an All-Reduced hand-off vector
    ``[beta, code(rank 0, mode 0..N-1), code(rank 1, ...), ...]`` (nncp_gamma_publish):
    lowest mode first, then lowest rank -- every rank reads the same vector, so every
    rank raises the same error (grid.py:172-203 re-raises one worker's exception)."""
    for n in range(order):
        for r in range(nranks):
            code = int(vec[1 + r * order + n])
            if code:
                return n, code >> 32, code & 0xFFFFFFFF
    return None


# test hook: "rank:iteration:mode:kind:row" makes that rank's update report a failure
# (kind 1 = BppCyclingError, 2 = singular) so the cross-rank hand-off can be exercised
# on real kernels; eager sweeps only.  Never set outside tests.
_FAULT_ENV = "NNCP_TEST_INJECT_FAULT"


def _state_arena(parts, dev):
    """One zeroed device allocation holding every (shape, dtype) of ``parts`` at 256-byte
    aligned offsets; returns (the byte buffer, typed views in order)."""
    offs, nbytes = [], 0
    for shape, dtype in parts:
        offs.append(nbytes)
        size = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        nbytes += (size + 255) // 256 * 256
    buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=dev)
    views = []
    for (shape, dtype), off in zip(parts, offs):
        esize = torch.empty((), dtype=dtype).element_size()
        count = int(np.prod(shape))
        views.append(buf[off:off + count * esize].view(dtype).view(shape))
    return buf, views


class _Engine:
    """One execution context (one GPU, or one simulated worker) of the SPMD program."""

    def __init__(self, x_local: torch.Tensor, local_dims, global_dims, cfg: RunConfig, coll, layout=None,
                 timing: bool = True, warn_negative: bool = False):
        self.x = x_local
        self.dims = tuple(int(d) for d in local_dims)
        self.global_dims = tuple(int(d) for d in global_dims)
        self.cfg = cfg
        self.coll = coll
        self.layout = layout
        self.N = len(self.dims)
        self.R = int(cfg.rank)
        self.algo = _lib.ALGO_CODES.get(cfg.algorithm, 0)
        dev = x_local.device
        self.dev = dev
        if layout is None:
            self.owned_rows = [slice(0, d) for d in self.global_dims]
            self.slice_rows = [slice(0, d) for d in self.global_dims]
            self.owned_parts = [block_partition(d, 1) for d in self.dims]
        else:
            self.owned_rows = list(layout.owned_rows)
            self.slice_rows = list(layout.slice_rows)
            self.owned_parts = list(layout.owned_parts)
        self.n_owned = [s.stop - s.start for s in self.owned_rows]
        f64 = dict(dtype=torch.float64, device=dev)
        self.lib = _lib.load()
        self.report = RunReport()
        self.timer = _EventTimer(timing)
        self._wall0 = time.perf_counter()
        # capture stream created before the first read-back below: torch's first Stream()
        # builds its stream pool (~40 ms in a fresh process, measured), which then overlaps
        # an asynchronous tensor upload instead of following it
        self.capture_stream = torch.cuda.Stream() if cfg.cuda_graph is not False else None
        # init row (driver.py:338-345): ||X||^2 of the local block, in the same read also
        # min x (negative-entry warning), max |x| and the smallest nonzero |x| -- the facts
        # the "auto" MTTKRP engine choice needs before the tensor is sliced
        self.scal = torch.zeros(7, **f64)     # beta, gamma, alpha, beta0, min x, max |x|, min nonzero |x|
        self.timer.start()
        norm_ws = Workspace(1 << 20)
        # when the cost model would slice this tensor, the row maxima of the slicing come
        # out of the same read of X as the facts (nncp_norm_rowmax; the planes follow
        # once the facts allow slicing), else the plain norm pass
        plan0, may_slice = _engine_plan(self.dims, cfg, dev)
        pre = None
        if may_slice and x_local.numel() > 0 and cfg.algorithm != "ucp":
            pre = SlicedTensor(x_local, self.dims, plan0.split, cfg.mttkrp_levels, defer=True)
            pre.norm_rowmax(x_local, _lib.vp(self.scal.data_ptr() + 16), _lib.vp(self.scal.data_ptr() + 32), norm_ws)
        else:
            _lib.check(self.lib.nncp_norm_squared_min(_lib.ptr(x_local), x_local.numel(),
                                                      _lib.vp(self.scal.data_ptr() + 16),
                                                      _lib.vp(self.scal.data_ptr() + 32), norm_ws.ptr,
                                                      norm_ws.nbytes, _lib.stream_handle()))
        self.timer.mark("Error")
        sc = self.scal.tolist()
        self.facts = TensorFacts(sc[2], sc[4], sc[5], sc[6])
        # (the buffer already held counts as available memory)
        held = pre.buf.numel() if pre is not None else 0
        self.plan, use_sliced = _engine_plan(self.dims, cfg, dev, extra_bytes=-held, facts=self.facts)
        self.sliced = None
        if use_sliced and pre is not None and pre.split == self.plan.split:
            pre.finish_planes(x_local)
            self.sliced = pre
        elif use_sliced:
            self.sliced = SlicedTensor(x_local, self.dims, self.plan.split, cfg.mttkrp_levels)
        del pre
        ws_bytes = self.plan.workspace_bytes()
        if self.sliced is not None:
            ws_bytes = max(ws_bytes, self.plan.sliced_workspace_bytes(self.sliced.levels))
        self.ws = Workspace(ws_bytes)
        self.ctx = DimTreeContext(self.plan, workspace=self.ws, sliced=self.sliced)
        # partials -> "MTTKRP", TTVs -> "MultiTTV" (the reference's recorder, dimtree.py:209-233)
        self.ctx.marker = self.timer.mark if timing else None
        R, N = self.R, self.N
        self.nsq = torch.zeros(R, **f64)
        # grid runs over NCCL: norm + Gram All-Reduces merged into one (DistCollectives)
        self.merge_norm_gram = bool(getattr(coll, "merge_norm_gram", False))
        self.graw = torch.zeros((R, R), **f64) if self.merge_norm_gram else None
        # driver.py:571-573: the negative-entry warning, from the initial norm pass
        self.warn_negative = bool(warn_negative) and cfg.algorithm != "ucp"
        self.status = torch.zeros((N, _lib.STATUS_WORDS), dtype=torch.int32, device=dev)
        _lib.check(self.lib.nncp_status_reset_n(_lib.ptr(self.status), N, _lib.stream_handle()))
        # end-of-sweep hand-off (grid.py:172-203): [beta, failure code per (rank, mode)].
        # The last update writes beta into slot 0, nncp_gamma_publish zeroes the code slots,
        # writes this rank's and resets the status words; ONE SUM All-Reduce (the
        # reference's beta All-Reduce, driver.py:429) then gives every rank every failure,
        # so all ranks raise the same error in the same iteration instead of one rank
        # leaving the others blocked in the next collective.
        self.nranks = layout.grid.total if layout is not None else 1
        self.me = layout.rank if layout is not None else 0
        self.xvec = torch.zeros(1 + self.nranks * N, **f64)
        self.masks = torch.zeros(2 * N, dtype=torch.int32, device=dev)
        # BPP: every owned row's final passive set, the next outer iteration's start
        # (nncp_update_ex; same final solve as the reference's cold start, fewer passes)
        fault = os.environ.get(_FAULT_ENV)
        self.fault = tuple(int(v) for v in fault.split(":")) if fault else None
        self.mbar = torch.empty((max(self.dims), R), **f64)
        self.hhat = torch.empty((max(max(self.n_owned), 1), R), **f64)
        # the state one sweep hands to the next -- factors, lambda, Grams, BPP passive
        # sets -- lives in ONE allocation, so a single copy snapshots it (run-ahead replays)
        bpp = cfg.algorithm == "bpp" and cfg.bpp_warm_start
        parts = [((self.n_owned[n], R), torch.float64) for n in range(N)]
        if coll.parallel:
            parts += [((self.dims[n], R), torch.float64) for n in range(N)]
        parts += [((R,), torch.float64), ((N, R, R), torch.float64)]
        if bpp:
            # passive sets, then the block nncp_bpp_prepare fills with S and S^-1
            parts += [((int(self.lib.nncp_bpp_sets_words(self.n_owned[n], R)),), torch.int64) for n in range(N)]
        self.state, views = _state_arena(parts, dev)
        self.state_backup = torch.empty_like(self.state)
        self.owned = views[:N]
        self.shared = views[N:2 * N] if coll.parallel else self.owned
        k = 2 * N if coll.parallel else N
        self.lam, self.grams = views[k], views[k + 1]
        self.lam.fill_(1.0)
        self.bpp_sets = views[k + 2:] if bpp else None
        # BPP: S and S^-1 of mode n need only the Grams, so they are formed on a second
        # stream while mode n's MTTKRP runs (fork / join events, captured into the graph)
        # (NNCP_BPP_PREPARE=0: formed inside the update, for A/B measurements)
        self.prep_stream = torch.cuda.Stream() if bpp and os.environ.get("NNCP_BPP_PREPARE") != "0" else None
        self.host_scal, self.host_xvec, self.host_masks = self._host_buffers()
        # stateful rules (updaters.py:56-68): per-mode ADMM dual / Nesterov centre
        rows_max = max(max(self.n_owned), 1)
        if cfg.algorithm in ("admm", "nes"):
            self.cur = torch.empty((rows_max, R), **f64)
            if cfg.algorithm == "admm":
                self.runner = AdmmRunner(rows_max, R, dev, self.ws)
                self.admm_dual = [torch.zeros((self.n_owned[n], R), **f64) for n in range(N)]
            else:
                self.runner = NesterovRunner(rows_max, R, dev, self.ws)
                self.nes_prev = [None] * N
        self.graphs = []            # [(CUDA graph of one sweep, its timing marks, its read-back buffers)]
        self.graph_failed = False
        self.graph_kernels = 0      # library kernels captured in the sweep graph
        self.graph_replays = 0

    # -- small wrappers -------------------------------------------------------
    def _st(self):
        return _lib.stream_handle()

    def _cmark(self, category):
        """Timer mark after a collective; a single context's collectives are no-ops, and
        an event-record node costs ~1-2 us of GPU timeline, so none is recorded for them."""
        if self.coll.parallel:
            self.timer.mark(category)

    def _gather(self, n):
        if self.coll.parallel:
            self.coll.all_gather(n, self.owned[n], self.owned_parts[n], out=self.shared[n])

    # -- initialisation (driver.py:338-373) -----------------------------------
    def initialise(self):
        lib, st, R = self.lib, self._st(), self.R
        self.report.begin_row()
        wall0 = self._wall0          # the norm pass ran in __init__ (it picks the engine)
        alpha_t = self.scal[2:3]
        self.coll.all_reduce(alpha_t)
        self._cmark("AllReduce")
        self.alpha = float(alpha_t.item())
        if self.warn_negative and self.facts.signed:
            warnings.warn("tensor has negative entries; nonnegative model will not fit")
        if self.alpha <= 0.0:
            raise ValueError("zero tensor has no relative error")
        cfg = self.cfg
        for n, size in enumerate(self.global_dims):
            if cfg.initial_factors is not None:
                full = cfg.initial_factors.factors[n]
                full = full.detach().cpu().numpy() if isinstance(full, torch.Tensor) else np.asarray(full, np.float64)
                if full.shape != (size, R):
                    raise ValueError(f"initial factor {n} has shape {full.shape}")
            else:
                full = init_factor(cfg.seed, n, size, R)
            self.owned[n].copy_(torch.from_numpy(np.ascontiguousarray(full[self.owned_rows[n]])))
            if self.coll.parallel:
                self.shared[n].copy_(torch.from_numpy(np.ascontiguousarray(full[self.slice_rows[n]])))
        if cfg.initial_factors is not None:
            lam0 = cfg.initial_factors.lam
            lam0 = lam0.detach().cpu().numpy() if isinstance(lam0, torch.Tensor) else np.asarray(lam0, np.float64)
            self.lam.copy_(torch.from_numpy(np.ascontiguousarray(lam0)))
        self.timer.mark("Error")
        for n in range(self.N):
            _lib.check(lib.nncp_gram(_lib.ptr(self.owned[n]), self.n_owned[n], R, _lib.ptr(self.grams[n]),
                                     self.ws.ptr, self.ws.nbytes, st))
            self.timer.mark("Gram")
            self.coll.all_reduce(self.grams[n])
            self._cmark("AllReduce")
            self._gather(n)
            self._cmark("AllGather")
        self.report.split_mode = self.plan.split if cfg.use_dimtree else None
        # initial model error from an out-of-band last-mode MTTKRP (driver.py:362-373);
        # the reference uses the einsum oracle here, the device reuses the tree kernels
        calls = self.ctx.partial_calls
        mb = self.mbar[: self.dims[-1]]
        self.ctx.mttkrp_last_mode(self.x, self.shared, out=mb)
        self.ctx.partial_calls = calls
        self.timer.mark("MTTKRP")
        _lib.check(lib.nncp_inner(_lib.ptr(mb), _lib.ptr(self.shared[-1]), _lib.ptr(self.lam), self.dims[-1], R,
                                  _lib.vp(self.scal.data_ptr() + 24), self.ws.ptr, self.ws.nbytes, st))
        self.timer.mark("Error")
        self.coll.all_reduce(self.scal[3:4])
        self._cmark("AllReduce")
        _lib.check(lib.nncp_gamma(_lib.ptr(self.grams), self.N, R, _lib.ptr(self.lam),
                                  _lib.vp(self.scal.data_ptr() + 8), st))
        self.timer.mark("Error")
        beta0, gamma0 = self.scal[3].item(), self.scal[1].item()
        self.report.errors = [_eps_from_terms(self.alpha, beta0, gamma0)]
        self.timer.collect(self.report.rows[-1])
        self.report.row_wall[-1] = time.perf_counter() - wall0
        self.report.row_words[-1] = self.coll.counters.total_words()

    # -- one outer iteration (driver.py:380-433), launches only ----------------
    def _sweep(self):
        lib, st, R, N = self.lib, self._st(), self.R, self.N
        cfg = self.cfg
        if cfg.use_dimtree:
            self.ctx.begin_iteration()
        # a single context hands the tree's column-major result to the fused update as
        # is (m_ld); grids need row blocks for the Reduce-Scatter
        in_place = not self.coll.parallel and cfg.algorithm in FUSED_ALGORITHMS
        published = False
        for n in range(N):
            mb = self.mbar[: self.dims[n]]
            m_ld = 0
            rows_n = self.n_owned[n]
            prep_done = self._bpp_prepare(n) if self.prep_stream is not None and rows_n > 0 else None
            fused_tail = in_place and R <= 32 and 1 <= rows_n and rows_n * R * R <= FUSED_TAIL_MAX
            grouped = None
            if in_place:
                # a sliced root partial may hand its split-K groups to the update (one
                # launch fewer: nncp_update_grouped sums them while loading the rows)
                defer = cfg.use_dimtree and not fused_tail and cfg.algorithm in ("mu", "hals", "bpp")
                temp = (self.ctx.mttkrp(self.x, self.shared, n, rows=False, defer_groups=defer) if cfg.use_dimtree
                        else self.ctx.mttkrp_direct(self.x, self.shared, n, rows=False))
                if isinstance(temp, DeferredPartial):
                    grouped, m_ld = temp, self.dims[n]
                else:
                    mb, m_ld = temp.data, self.dims[n]
            elif cfg.use_dimtree:
                self.ctx.mttkrp(self.x, self.shared, n, out=mb)
            else:
                self.ctx.mttkrp_direct(self.x, self.shared, n, out=mb)
            self.timer.mark("MTTKRP")
            m_owned = self.coll.reduce_scatter(n, mb, self.owned_parts[n])
            self._cmark("ReduceScatter")
            if prep_done is not None:
                torch.cuda.current_stream().wait_event(prep_done)   # join: S, S^-1 ready
            last = n == N - 1
            if fused_tail:
                # small single-context block: the update kernel's last CTA also normalises,
                # forms the Gram (and for the last mode gamma + the status hand-off)
                _lib.check(lib.nncp_update_normalize(
                    self.algo, _lib.ptr(self.grams), N, n, R, _lib.ptr(m_owned), _lib.ptr(self.owned[n]),
                    _lib.ptr(self.lam), rows_n, _lib.ptr(self.hhat), _lib.ptr(self.nsq),
                    _lib.ptr(self.xvec) if last else None, _lib.ptr(self.status[n]), 1e-16,
                    _lib.ptr(self.bpp_sets[n]) if self.bpp_sets else None, m_ld, _lib.ptr(self.grams[n]),
                    _lib.vp(self.scal.data_ptr() + 8) if last else None, _lib.ptr(self.status), N,
                    _lib.vp(self.xvec.data_ptr() + 8), self.nranks * N, self.me * N, _lib.ptr(self.masks),
                    self.ws.ptr, self.ws.nbytes, st))
                self.timer.mark("NNLS")
                published = published or last
                continue
            if grouped is not None:
                _lib.check(lib.nncp_update_grouped(self.algo, _lib.ptr(self.grams), N, n, R, grouped.ptr, m_ld,
                                                   grouped.groups, grouped.gstride, _lib.ptr(self.owned[n]),
                                                   _lib.ptr(self.lam), rows_n, _lib.ptr(self.hhat),
                                                   _lib.ptr(self.nsq), _lib.ptr(self.xvec) if last else None,
                                                   _lib.ptr(self.status[n]), 1e-16,
                                                   _lib.ptr(self.bpp_sets[n]) if self.bpp_sets else None,
                                                   self.ws.ptr, self.ws.nbytes, st))
            elif cfg.algorithm in FUSED_ALGORITHMS:
                _lib.check(lib.nncp_update_ex(self.algo, _lib.ptr(self.grams), N, n, R, _lib.ptr(m_owned),
                                              _lib.ptr(self.owned[n]), _lib.ptr(self.lam), self.n_owned[n],
                                              _lib.ptr(self.hhat), _lib.ptr(self.nsq),
                                              _lib.ptr(self.xvec) if last else None, _lib.ptr(self.status[n]),
                                              1e-16, _lib.ptr(self.bpp_sets[n]) if self.bpp_sets else None,
                                              m_ld, self.ws.ptr, self.ws.nbytes, st))
            else:
                self._iterative_update(n, m_owned, last)
            self.timer.mark("NNLS")
            if self.fault is not None and self.fault[:3] == (self.me, len(self.report.errors), n):
                self.status[n, 3] = self.fault[3]
                self.status[n, 2] = self.fault[4]
            if self.merge_norm_gram:
                # one All-Reduce of the unnormalised Gram: its diagonal is nsq
                _lib.check(lib.nncp_gram(_lib.ptr(self.hhat), self.n_owned[n], R, _lib.ptr(self.graw),
                                         self.ws.ptr, self.ws.nbytes, st))
                self.timer.mark("Gram")
                self.coll.all_reduce(self.graw)
                self._cmark("AllReduce")
                _lib.check(lib.nncp_normalize_from_gram(_lib.ptr(self.hhat), _lib.ptr(self.graw), self.n_owned[n],
                                                        R, _lib.ptr(self.owned[n]), _lib.ptr(self.lam),
                                                        _lib.ptr(self.grams[n]), st))
                self.timer.mark("NNLS")
            elif last and not self.coll.parallel:
                # a single context: the last normalisation also computes gamma and hands
                # the status words off (nncp_gamma_publish folded in, one launch fewer)
                _lib.check(lib.nncp_normalize_gram_publish(
                    _lib.ptr(self.hhat), _lib.ptr(self.nsq), self.n_owned[n], R, _lib.ptr(self.owned[n]),
                    _lib.ptr(self.lam), _lib.ptr(self.grams[n]), self.ws.ptr, self.ws.nbytes, _lib.ptr(self.grams), N,
                    _lib.vp(self.scal.data_ptr() + 8), _lib.ptr(self.status), N, _lib.vp(self.xvec.data_ptr() + 8),
                    self.nranks * N, self.me * N, _lib.ptr(self.masks), st))
                self.timer.mark("Gram")
                published = True
            else:
                self.coll.all_reduce(self.nsq)
                self._cmark("AllReduce")
                _lib.check(lib.nncp_normalize_gram(_lib.ptr(self.hhat), _lib.ptr(self.nsq), self.n_owned[n], R,
                                                   _lib.ptr(self.owned[n]), _lib.ptr(self.lam),
                                                   _lib.ptr(self.grams[n]), self.ws.ptr, self.ws.nbytes, st))
                self.timer.mark("Gram")
                self.coll.all_reduce(self.grams[n])
                self._cmark("AllReduce")
            self._gather(n)
            self._cmark("AllGather")
        if not published:
            _lib.check(lib.nncp_gamma_publish(_lib.ptr(self.grams), N, R, _lib.ptr(self.lam),
                                              _lib.vp(self.scal.data_ptr() + 8), _lib.ptr(self.status), N,
                                              _lib.vp(self.xvec.data_ptr() + 8), self.nranks * N, self.me * N,
                                              _lib.ptr(self.masks), st))
            self.timer.mark("Error")
        self.coll.all_reduce(self.xvec, words=1)      # beta + every rank's status codes
        self._cmark("AllReduce")
        self.host_xvec.copy_(self.xvec, non_blocking=True)
        self.host_scal.copy_(self.scal[0:2], non_blocking=True)
        self.host_masks.copy_(self.masks, non_blocking=True)
        self.timer.mark("Error")

    def _bpp_prepare(self, n):
        """Fork: BPP's S and S^-1 for mode n (nncp_bpp_prepare) on the side stream, after
        everything queued so far (the Grams of the modes before n); returns the join event."""
        fork = torch.cuda.Event()
        fork.record()
        self.prep_stream.wait_event(fork)
        with torch.cuda.stream(self.prep_stream):
            _lib.check(self.lib.nncp_bpp_prepare(_lib.ptr(self.grams), self.N, n, self.R,
                                                 _lib.ptr(self.bpp_sets[n]), self.n_owned[n], self._st()))
        done = torch.cuda.Event()
        done.record(self.prep_stream)
        return done

    def _hook(self, t, op):
        return self.coll.all_reduce(t, op)

    def _iterative_update(self, n, m_owned, last):
        """ADMM / NES for mode n (updaters.py:173-281) through the collective hook."""
        lib, st, R = self.lib, self._st(), self.R
        rows = self.n_owned[n]
        cur = self.cur[:rows]
        _lib.check(lib.nncp_scale_columns(_lib.ptr(self.owned[n]), _lib.ptr(self.lam), rows, R, _lib.ptr(cur), st))
        spack = _SPack(self.grams, self.N, n)
        try:
            if self.cfg.algorithm == "admm":
                x, _ = self.runner.run(spack, m_owned, cur, self.admm_dual[n], self._hook, status=self.status[n],
                                       defer_errors=True)
            else:
                xstar = self.nes_prev[n] if self.nes_prev[n] is not None else cur
                x, _ = self.runner.run(spack, m_owned, cur, xstar, self._hook)
                if self.nes_prev[n] is None:
                    self.nes_prev[n] = torch.empty_like(x[:rows])
                self.nes_prev[n].copy_(x[:rows])
        except Exception as exc:
            raise RuntimeError(f"NNLS update failed at iteration {len(self.report.errors)}, mode {n + 1}") from exc
        hh = self.hhat[:rows]
        hh.copy_(x[:rows])
        _lib.check(lib.nncp_colsumsq(_lib.ptr(hh), rows, R, _lib.ptr(self.nsq), self.ws.ptr, self.ws.nbytes, st))
        if last:
            _lib.check(lib.nncp_inner(_lib.ptr(m_owned), _lib.ptr(hh), None, rows, R, _lib.ptr(self.xvec),
                                      self.ws.ptr, self.ws.nbytes, st))

    # -- Nesterov outer extrapolation (driver.py:452-492) ----------------------------
    def _snapshot(self):
        self.prev_owned = [h.clone() for h in self.owned]
        self.prev_shared = [h.clone() for h in self.shared] if self.coll.parallel else self.prev_owned
        self.prev_lam = self.lam.clone()

    def _model_error(self, cand_shared, cand_owned, cand_lam):
        """driver.py:310-328 on device buffers."""
        lib, st, R, N = self.lib, self._st(), self.R, self.N
        mb = self.mbar[: self.dims[-1]]
        if self.cfg.use_dimtree:
            self.ctx.mttkrp_last_mode(self.x, cand_shared, out=mb)        # counts a tree partial, as the reference
        else:
            calls = self.ctx.partial_calls
            self.ctx.mttkrp_direct(self.x, cand_shared, N - 1, out=mb)
            self.ctx.partial_calls = calls
        sc = torch.zeros(2, dtype=torch.float64, device=self.dev)
        _lib.check(lib.nncp_inner(_lib.ptr(mb), _lib.ptr(cand_shared[-1]), _lib.ptr(cand_lam), self.dims[-1], R,
                                  _lib.ptr(sc), self.ws.ptr, self.ws.nbytes, st))
        self.coll.all_reduce(sc[0:1])
        grams = torch.zeros((N, R, R), dtype=torch.float64, device=self.dev)
        for n in range(N):
            _lib.check(lib.nncp_gram(_lib.ptr(cand_owned[n]), self.n_owned[n], R, _lib.ptr(grams[n]), self.ws.ptr,
                                     self.ws.nbytes, st))
            self.coll.all_reduce(grams[n])
        _lib.check(lib.nncp_gamma(_lib.ptr(grams), N, R, _lib.ptr(cand_lam), _lib.vp(sc.data_ptr() + 8), st))
        beta, gamma = sc.cpu().tolist()
        return _eps_from_terms(self.alpha, beta, gamma)

    def _nes_accelerate(self, it, eps):
        lib, st, R, N = self.lib, self._st(), self.R, self.N
        step = float(it) ** (1.0 / N)

        def extrap(cur, prev):
            out = torch.empty_like(cur)
            _lib.check(lib.nncp_extrapolate(_lib.ptr(cur), _lib.ptr(prev), cur.numel(), step, _lib.ptr(out), st))
            return out

        cand_owned = [extrap(h, hp) for h, hp in zip(self.owned, self.prev_owned)]
        cand_shared = ([extrap(h, hp) for h, hp in zip(self.shared, self.prev_shared)] if self.coll.parallel
                       else cand_owned)
        cand_lam = extrap(self.lam, self.prev_lam)
        cand_eps = self._model_error(cand_shared, cand_owned, cand_lam)
        if not cand_eps < eps:
            return
        nsq = torch.zeros((N, R), dtype=torch.float64, device=self.dev)
        for n in range(N):
            _lib.check(lib.nncp_colsumsq(_lib.ptr(cand_owned[n]), self.n_owned[n], R, _lib.ptr(nsq[n]), self.ws.ptr,
                                         self.ws.nbytes, st))
        self.coll.all_reduce(nsq)
        for n in range(N):
            _lib.check(lib.nncp_normalize_gram(_lib.ptr(cand_owned[n]), _lib.ptr(nsq[n]), self.n_owned[n], R,
                                               _lib.ptr(self.owned[n]), None, None, self.ws.ptr, self.ws.nbytes, st))
            if self.coll.parallel:
                _lib.check(lib.nncp_normalize_gram(_lib.ptr(cand_shared[n]), _lib.ptr(nsq[n]), self.dims[n], R,
                                                   _lib.ptr(self.shared[n]), None, None, self.ws.ptr,
                                                   self.ws.nbytes, st))
        _lib.check(lib.nncp_nes_lambda(_lib.ptr(cand_lam), _lib.ptr(nsq), N, R, _lib.ptr(self.lam), st))
        for n in range(N):
            _lib.check(lib.nncp_gram(_lib.ptr(self.owned[n]), self.n_owned[n], R, _lib.ptr(self.grams[n]),
                                     self.ws.ptr, self.ws.nbytes, st))
            self.coll.all_reduce(self.grams[n])

    def _finish_iteration(self, it, host=None, done=None):
        """Warnings, the failure hand-off and eps of sweep ``it`` from its read-back buffers
        (``host``; the eager buffers by default) once ``done`` (default: the stream) is reached."""
        host_scal, host_xvec, host_masks = host if host is not None else (self.host_scal, self.host_xvec,
                                                                          self.host_masks)
        if done is not None:
            done.synchronize()
        else:
            torch.cuda.current_stream().synchronize()
        masks = host_masks.tolist()
        for n in range(self.N):
            warn_for_status(masks[2 * n], masks[2 * n + 1], self.cfg.algorithm)
        vec = host_xvec.tolist()
        fail = first_failure(vec, self.nranks, self.N)
        if fail is not None:
            n, kind, row = fail
            torch.cuda.current_stream().synchronize()     # a run-ahead replay may still be in flight
            try:
                raise_for_code(kind, row)
            except Exception as exc:
                raise RuntimeError(f"NNLS update failed at iteration {it}, mode {n + 1}") from exc
        return _eps_from_terms(self.alpha, vec[0], host_scal[1].item())

    def iterate(self, count: int = None):
        """Run up to ``count`` more outer iterations (default: the rest of max_iters)."""
        cfg = self.cfg
        errors = self.report.errors
        capturable = ((not self.coll.parallel or getattr(self.coll, "capturable", False))
                      and cfg.algorithm in FUSED_ALGORITHMS)
        use_graph = (capturable and (cfg.cuda_graph is None or bool(cfg.cuda_graph))) and self.fault is None
        done = len(errors) - 1
        stop = cfg.max_iters if count is None else min(cfg.max_iters, done + count)
        ahead = None        # the replay launched for iteration it+1 before iteration it's stop test
        for it in range(done + 1, stop + 1):
            self.report.begin_row()
            wall0 = time.perf_counter()
            if use_graph and not self.graphs and it > 1 and not self.graph_failed:
                self._capture_graphs()
            if self.graphs:
                cur = ahead if ahead is not None else self._launch_replay()
                # run ahead: queue sweep it+1 behind sweep it, so the GPU works while the
                # host waits for eps_it; undone (state restored from the replay's own
                # snapshot) if sweep it turns out to be the last
                ahead = self._launch_replay() if it + 1 <= stop else None
                marks, host, done_ev = cur
                eps = self._finish_iteration(it, host, done_ev)
                self.coll.counters.add(self.graph_comm)
                if cfg.use_dimtree:
                    self.ctx.partial_calls += 2
                self.timer.collect_marks(marks, self.report.rows[-1])   # sweep it+1 runs meanwhile
            else:
                self.timer.start()
                if cfg.algorithm == "nes":
                    self._snapshot()
                self._sweep()
                eps = self._finish_iteration(it)
                self.timer.collect(self.report.rows[-1])
            errors.append(eps)
            if cfg.algorithm == "nes":
                self._nes_accelerate(it, eps)
            self.report.row_wall[-1] = time.perf_counter() - wall0
            self.report.row_words[-1] = self.coll.counters.total_words() - sum(self.report.row_words[:-1])
            if eps <= cfg.tol:
                self.report.converged = True
                if ahead is not None:
                    self.state.copy_(self.state_backup)     # undo the run-ahead sweep
                    torch.cuda.current_stream().synchronize()
                break
        self.report.tree_partial_calls = self.ctx.partial_calls if cfg.use_dimtree else 0

    def _launch_replay(self):
        """Replay the next copy of the sweep graph; (its timing marks, its read-back
        buffers, an event marking its end)."""
        g, marks, host = self.graphs[self.graph_replays % len(self.graphs)]
        g.replay()
        done = torch.cuda.Event()
        done.record()
        self.graph_replays += 1
        return marks, host, done

    @property
    def graph(self):
        return self.graphs[0][0] if self.graphs else None

    def set_timing(self, enabled: bool):
        """Turn the per-category CUDA events on or off for the following sweeps (the
        sweep graphs are re-captured without / with their event-record nodes; each
        costs ~1-2 us of GPU timeline, which matters for the smallest tensors)."""
        enabled = bool(enabled)
        if enabled == self.timer.enabled:
            return
        self.timer.enabled = enabled
        self.ctx.marker = self.timer.mark if enabled else None
        self.graphs = []

    def _capture_graphs(self):
        """Two copies of the sweep graph, each with its own timing events and pinned
        read-back buffers, replayed alternately: sweep i+1 is launched before the host
        reads sweep i's error (run-ahead), so the GPU never idles on the stop test."""
        graphs = []
        for _ in range(2):
            cap = self._capture()
            if cap is None:
                return
            graphs.append(cap)
        self.graphs = graphs

    def _capture(self):
        """Record one sweep as a CUDA graph (all buffers already allocated by sweep 1);
        returns (graph, timing marks) or None when capture failed (eager from then on)."""
        calls = self.ctx.partial_calls
        launches0 = self.lib.nncp_launch_count()
        comm0 = self.coll.counters.snapshot()
        g = torch.cuda.CUDAGraph()
        side = self.capture_stream or torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        # capture_begin/end directly: torch.cuda.graph's context manager also empties
        # the allocator caches (device and pinned host), which this capture does not
        # need -- every buffer of the sweep already exists after sweep 1
        # each captured copy D2H-copies into its own pinned buffers: a run-ahead replay of
        # the other copy must not overwrite what the host has not read yet
        host = self._host_buffers()
        self.host_scal, self.host_xvec, self.host_masks = host
        try:
            torch.cuda.synchronize()
            with torch.cuda.stream(side):
                g.capture_begin()
                try:
                    # snapshot of the incoming state (one memcpy node): a replay launched
                    # ahead of the previous sweep's stop test can be undone
                    self.state_backup.copy_(self.state)
                    self.timer.begin_capture()
                    self._sweep()
                    self.timer.end_capture()
                finally:
                    g.capture_end()
        except Exception as exc:  # noqa: BLE001  (stay on the eager path, still correct)
            self.timer.capturing = False
            warnings.warn(f"CUDA graph capture failed, continuing without graphs: {exc}")
            torch.cuda.current_stream().wait_stream(side)
            self.ctx.partial_calls = calls
            self.coll.counters.restore(comm0)
            self.graph_failed = True
            self.graphs = []
            return None
        torch.cuda.current_stream().wait_stream(side)
        self.ctx.partial_calls = calls
        self.graph_kernels = int(self.lib.nncp_launch_count() - launches0)
        # capturing ran no collective: every replay adds the captured calls and words
        # (grid.py:60-93 tallies per call)
        self.graph_comm = self.coll.counters.since(comm0)
        self.coll.counters.restore(comm0)
        return g, self.timer.graph_marks, host

    def _host_buffers(self):
        pin = dict(pin_memory=True)
        return (torch.zeros(2, dtype=torch.float64, **pin),
                torch.zeros(1 + self.nranks * self.N, dtype=torch.float64, **pin),
                torch.zeros(2 * self.N, dtype=torch.int32, **pin))

    def model_host(self):
        return [h.detach().cpu().numpy() for h in self.owned], self.lam.detach().cpu().numpy()


def _warn_if_negative(x: DenseTensor, cfg: RunConfig):
    """driver.py:571-573 (min over the device copy)."""
    if cfg.algorithm == "ucp":
        return
    d = x.data
    lo = float(torch.min(d).item()) if isinstance(d, torch.Tensor) else float(np.min(d))
    if lo < 0.0:
        warnings.warn("tensor has negative entries; nonnegative model will not fit")


def run_local(x_local: torch.Tensor, local_dims, global_dims, cfg: RunConfig, coll=None, layout=None,
              timing: bool = True, warn_negative: bool = False):
    """Run the SPMD program on one execution context; returns (engine, report)."""
    eng = _Engine(x_local, local_dims, global_dims, cfg, coll or IdentityCollectives(), layout, timing,
                  warn_negative=warn_negative)
    eng.initialise()
    eng.iterate()
    eng.report.counters = eng.coll.counters
    return eng, eng.report


def nncp_sequential(x: DenseTensor, cfg: RunConfig) -> RunReport:
    """Single-GPU NNCP (driver.py:495-505); the tensor is copied to HBM once if needed."""
    cfg.validate(x.order)
    if cfg.grid is not None and int(np.prod(cfg.grid)) != 1:
        raise ValueError("sequential driver got a nontrivial grid; use nncp_parallel")
    if not x.on_device:
        _reserve_sliced(x.dims, cfg)
    xd = x.to_device()
    # the negative-entry warning comes from the engine's first pass over the tensor
    eng, rep = run_local(xd.data, x.dims, x.dims, cfg, warn_negative=True)
    owned, lam = eng.model_host()
    rep.model = FactorSet(owned, lam)
    return rep


def nncp_parallel(x: DenseTensor, cfg: RunConfig) -> RunReport:
    """Grid-parallel NNCP (driver.py:508-531).

    Inside a torch.distributed job whose world size equals prod(grid), each
    process runs its grid block on its own GPU (NCCL collectives) and every
    rank returns the merged report.  Otherwise the grid is simulated by worker
    threads on the local GPU with rank-ordered, bitwise-reproducible
    collectives (the reference's execution model, grid.py:172-203).

    ``x`` is a DenseTensor (host, pinned, memory-mapped or device-resident) or
    the path of an NNCP tensor file; every rank copies only its own block
    (driver.py:233-236): from a file it reads just the block's byte ranges,
    from a device tensor it slices in HBM, from host memory it copies the block.
    """
    if isinstance(x, (str, os.PathLike)):
        from .tensor_io import read_tensor_dims

        dims = read_tensor_dims(x)
    else:
        dims = x.dims
    cfg.validate(len(dims))
    if cfg.grid is None:
        raise ValueError("parallel driver needs a grid shape")
    for n, (i, p) in enumerate(zip(dims, cfg.grid)):
        if p > i:
            raise ValueError(f"grid dim {p} exceeds tensor dim {i} in mode {n + 1}; "
                             "every worker must hold a nonempty tensor block")
    grid = Grid(cfg.grid)
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == grid.total:
        return _parallel_dist(x, dims, cfg, grid)
    if isinstance(x, (str, os.PathLike)):
        from .tensor_io import read_tensor

        x = read_tensor(x)
    return _parallel_threads(x, cfg, grid)


def local_block(x, layout: RankLayout) -> torch.Tensor:
    """This rank's tensor block in HBM, flat and mode-1 fastest, never materialising
    more than the block on the host: file -> byte-range reads; device tensor -> a
    slice copy in HBM; host array -> the block's elements only."""
    offs = [s.start for s in layout.slice_rows]
    if isinstance(x, (str, os.PathLike)):
        from .tensor_io import read_tensor_block

        return as_device(read_tensor_block(x, offs, layout.local_dims))
    if x.on_device:
        # reversed-dims C view of the F-ordered buffer: index [i_N, ..., i_1]; always a
        # fresh allocation (a contiguous slice would be an offset view, not 16-byte aligned)
        view = x.data.view(tuple(reversed(x.dims)))[tuple(reversed(layout.slice_rows))]
        out = torch.empty(view.shape, dtype=torch.float64, device=x.data.device)
        out.copy_(view)
        return out.view(-1)
    arr = x.as_array()[tuple(layout.slice_rows)]
    return as_device(np.asarray(arr).ravel(order="F"))


def _parallel_threads(x: DenseTensor, cfg: RunConfig, grid: Grid) -> RunReport:
    tgrid = ThreadGrid(grid)
    results = [None] * grid.total
    failures = [None] * grid.total
    dev = torch.cuda.current_device()
    _warn_if_negative(x, cfg)

    def main(rank):
        try:
            torch.cuda.set_device(dev)
            layout = RankLayout(grid, rank, x.dims)
            coll = ThreadCollectives(tgrid, layout)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                xl = local_block(x, layout)       # on the worker's stream, ahead of its kernels
                eng, rep = run_local(xl, layout.local_dims, x.dims, cfg, coll, layout)
                owned, lam = eng.model_host()
            results[rank] = (rep, owned, lam, layout.owned_rows)
        except threading.BrokenBarrierError:
            pass
        except BaseException as exc:  # noqa: BLE001  (propagate to the caller)
            failures[rank] = exc
            tgrid.abort()

    threads = [threading.Thread(target=main, args=(r,), name=f"nncp-worker-{r}") for r in range(grid.total)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for exc in failures:
        if exc is not None:
            raise exc
    return _merge_reports(results, x.dims, cfg.rank)


def _parallel_dist(x, dims, cfg: RunConfig, grid: Grid) -> RunReport:
    import torch.distributed as dist

    rank = dist.get_rank()
    layout = RankLayout(grid, rank, dims)
    coll = DistCollectives(layout)
    xl = local_block(x, layout)
    if cfg.algorithm != "ucp":
        # driver.py:571-573 over the whole tensor: min of the blocks (an init-time
        # reduction outside the reference's counted collectives)
        lo = torch.min(xl).reshape(1).to(torch.float64)
        if coll.stage:
            lo = lo.cpu()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        if rank == 0 and float(lo.item()) < 0.0:
            warnings.warn("tensor has negative entries; nonnegative model will not fit")
    eng, rep = run_local(xl, layout.local_dims, dims, cfg, coll, layout)
    owned, lam = eng.model_host()
    gathered = [None] * grid.total
    dist.all_gather_object(gathered, (rep, owned, lam, layout.owned_rows))
    return _merge_reports(gathered, dims, cfg.rank)


def _merge_reports(results, dims, rank) -> RunReport:
    """driver.py:534-568: averaged seconds, summed words and counters, assembled model."""
    merged = RunReport()
    first = results[0][0]
    nworkers = len(results)
    merged.errors = list(first.errors)
    merged.split_mode = first.split_mode
    merged.converged = first.converged
    merged.tree_partial_calls = first.tree_partial_calls
    for rep, _, _, _ in results:
        if not np.allclose(rep.errors, first.errors, rtol=0, atol=1e-12):
            raise AssertionError("workers disagree on the error sequence")
    for k in range(len(first.rows)):
        merged.begin_row()
        for cat in CATEGORIES:
            merged.rows[k][cat] = sum(r.rows[k][cat] for r, _, _, _ in results) / nworkers
        merged.row_words[k] = sum(r.row_words[k] for r, _, _, _ in results)
        merged.row_wall[k] = sum(r.row_wall[k] for r, _, _, _ in results) / nworkers
    counters = CommCounters()
    for rep, _, _, _ in results:
        counters = counters.merged_with(rep.counters)
    merged.counters = counters
    factors = [np.zeros((i, rank)) for i in dims]
    for _, owned, _, rows in results:
        for n, (h, s) in enumerate(zip(owned, rows)):
            factors[n][s] = h
    merged.model = FactorSet(factors, results[0][2])
    return merged
