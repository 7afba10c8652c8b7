"""N-d processor grid and the three collectives of the NNCP step (reference: nncp/grid.py).

Grid semantics are the reference's (grid.py:129-170): rank = p_1 + P_1 p_2 + ...
(mode-1 coordinate fastest), the mode-n slice of a rank is every rank sharing
its n-th coordinate (sorted), tensor blocks and owned factor rows come from
``block_partition`` (first ``length % parts`` blocks get one extra row).

Three interchangeable collective backends sit behind one interface
(``all_reduce`` / ``reduce_scatter`` / ``all_gather``, the swap point the
reference documents at pkg/README.md:133-136):

* ``IdentityCollectives`` -- one context, every collective is the identity;
* ``DistCollectives``     -- one process per GPU over ``torch.distributed``
  (NCCL over NVLink/NVSwitch on the B200 box; gloo for the CPU tests), one
  global group plus one sub-group per mode slice;
* ``ThreadCollectives``   -- workers as threads in one process sharing the
  local GPU(s); rank-ordered device-side reductions, bitwise reproducible
  (what ``nncp_parallel`` uses when no process group is running).

Word counters follow CommCounters (grid.py:60-93): words_in = elements
entering the call, words_out = elements leaving it.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

__all__ = ["block_partition", "DistMap", "CommCounters", "Group", "Grid", "Worker", "IdentityCollectives",
           "DistCollectives", "ThreadCollectives", "ThreadGrid", "pin_nccl_environment"]


def block_partition(length: int, parts: int) -> "DistMap":
    """Balanced contiguous blocks; the first ``length % parts`` are one longer (grid.py:25-31)."""
    if length < 0 or parts < 1:
        raise ValueError(f"bad partition request: length={length}, parts={parts}")
    sizes = np.full(int(parts), int(length) // int(parts), dtype=np.int64)
    sizes[: int(length) % int(parts)] += 1
    return DistMap(sizes)


class DistMap:
    """A contiguous split of [0, total) into blocks (grid.py:34-57): ``lengths`` and
    the ``offsets`` of their starts (plus the end)."""

    __slots__ = ("lengths", "offsets")

    def __init__(self, lengths):
        arr = np.asarray(list(lengths), dtype=np.int64).reshape(-1)
        if (arr < 0).any():
            raise ValueError("block lengths must be nonnegative")
        self.lengths = tuple(int(v) for v in arr)
        self.offsets = tuple(int(v) for v in np.concatenate(([0], np.cumsum(arr))))

    parts = property(lambda self: len(self.lengths))
    total = property(lambda self: self.offsets[-1])
    max_length = property(lambda self: max(self.lengths, default=0))

    def block(self, k: int) -> slice:
        return slice(self.offsets[k], self.offsets[k + 1])


_TALLIES = ("calls", "words_in", "words_out", "seconds")


@dataclass
class CommCounters:
    """Per-rank collective tallies keyed by collective name (grid.py:60-93): calls,
    words entering / leaving each call, seconds.  Also snapshot / delta / re-add /
    restore for the CUDA-graph replays, which run captured collectives again."""

    calls: dict = field(default_factory=dict)
    words_in: dict = field(default_factory=dict)
    words_out: dict = field(default_factory=dict)
    seconds: dict = field(default_factory=dict)

    def _bump(self, name, calls, w_in, w_out, secs=0.0):
        for tally, v in zip(_TALLIES, (calls, w_in, w_out, secs)):
            d = getattr(self, tally)
            d[name] = d.get(name, 0.0 if tally == "seconds" else 0) + v

    def record(self, name: str, words_in: int, words_out: int, elapsed: float = 0.0):
        self._bump(name, 1, int(words_in), int(words_out), elapsed)

    def snapshot(self) -> dict:
        return {t: dict(getattr(self, t)) for t in _TALLIES[:3]}

    def since(self, snap: dict) -> dict:
        """The calls and words recorded after ``snap`` (one captured sweep's collectives)."""
        return {t: {k: v - snap[t].get(k, 0) for k, v in getattr(self, t).items()} for t in _TALLIES[:3]}

    def add(self, delta: dict):
        """Re-add a ``since`` delta (a CUDA-graph replay of the captured collectives)."""
        for name in delta["calls"]:
            self._bump(name, delta["calls"][name], delta["words_in"].get(name, 0), delta["words_out"].get(name, 0))

    def restore(self, snap: dict):
        """Back to ``snap`` (collectives recorded while capturing did not run)."""
        for t in _TALLIES[:3]:
            setattr(self, t, dict(snap[t]))

    def total_words(self) -> int:
        return sum(self.words_in.values()) + sum(self.words_out.values())

    def merged_with(self, other: "CommCounters") -> "CommCounters":
        out = CommCounters()
        for src in (self, other):
            for name in src.calls:
                out._bump(name, src.calls[name], src.words_in.get(name, 0), src.words_out.get(name, 0),
                          src.seconds.get(name, 0.0))
        return out


class Group:
    """An ascending rank set, each member's position in it, and its rendezvous
    (grid.py:116-126)."""

    def __init__(self, ranks):
        self.ranks = tuple(sorted(int(r) for r in ranks))
        self.index = dict(zip(self.ranks, range(len(self.ranks))))
        self.rendezvous = _Rendezvous(len(self.ranks))

    @property
    def size(self) -> int:
        return len(self.ranks)


class Grid:
    """P_1 x ... x P_N processor grid (grid.py:129-203).  A rank is the column-major
    (mode-1 fastest) linear index of its coordinate; the mode-n slice of a rank is
    every rank with the same n-th coordinate."""

    def __init__(self, shape):
        self.shape = tuple(int(p) for p in shape)
        if any(p < 1 for p in self.shape):
            raise ValueError(f"grid dims must be positive, got {self.shape}")
        self.total = int(np.prod(self.shape, dtype=np.int64))
        self.all_procs = Group(range(self.total))
        coords = np.array(np.unravel_index(np.arange(self.total), self.shape, order="F")).T.reshape(self.total, -1)
        self.slice_groups = [[Group(np.flatnonzero(coords[:, n] == c)) for c in range(pn)]
                             for n, pn in enumerate(self.shape)]

    def coord_of(self, rank: int):
        return tuple(int(c) for c in np.unravel_index(int(rank), self.shape, order="F"))

    def rank_of(self, coord) -> int:
        coord = tuple(int(c) for c in coord)
        if len(coord) != len(self.shape) or any(not 0 <= c < p for c, p in zip(coord, self.shape)):
            raise ValueError(f"coordinate {coord} outside grid {self.shape}")
        return int(np.ravel_multi_index(coord, self.shape, order="F"))

    def slice_group(self, mode: int, coord: int) -> Group:
        return self.slice_groups[mode][coord]

    def _groups(self):
        yield self.all_procs
        for per_mode in self.slice_groups:
            yield from per_mode

    def run(self, fn, *args):
        """Run ``fn(worker, *args)`` on every rank as a thread; the per-rank results
        (grid.py:172-203).  A failing rank breaks every rendezvous, so no rank is left
        waiting, and the first failure is raised in the caller."""
        self._workers = [Worker(r, self) for r in range(self.total)]
        out = [None] * self.total
        errors = [None] * self.total

        def body(w):
            try:
                out[w.rank] = fn(w, *args)
            except threading.BrokenBarrierError:
                return
            except BaseException as exc:  # noqa: BLE001  (propagate to the caller)
                errors[w.rank] = exc
                for g in self._groups():
                    g.rendezvous.abort()

        threads = [threading.Thread(target=body, args=(w,), name=f"worker-{w.rank}") for w in self._workers]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        first = next((e for e in errors if e is not None), None)
        if first is not None:
            raise first
        return out


def _fold(values, op):
    """Elementwise combination of the members' arrays in ascending rank order
    (grid.py:250-262), numpy on the host or torch on the device."""
    acc = values[0].clone() if isinstance(values[0], torch.Tensor) else np.array(values[0], copy=True)
    for v in values[1:]:
        if op == "sum":
            acc += v
        elif isinstance(acc, torch.Tensor):
            acc = torch.minimum(acc, v) if op == "min" else torch.maximum(acc, v)
        else:
            (np.minimum if op == "min" else np.maximum)(acc, v, out=acc)
    return acc


class Worker:
    """One rank inside ``Grid.run`` (grid.py:206-302): its coordinate, counters and the
    reference's collective calls on a ``Group``, bitwise reproducible (ascending rank
    order).  Host (numpy) payloads are combined on the host like the reference; CUDA
    tensors are combined on their device in the same order and returned on it.  The
    mailbox point-to-point pair ``send`` / ``recv`` (grid.py:224-237) is kept."""

    def __init__(self, rank: int, grid: "Grid"):
        self.rank = int(rank)
        self.grid = grid
        self.coord = grid.coord_of(self.rank)
        self.counters = CommCounters()
        self.recorder = None
        self._inbox = []
        self._inbox_cv = threading.Condition()

    def send(self, dst: int, payload):
        peer = self.grid._workers[dst]
        with peer._inbox_cv:
            peer._inbox.append((self.rank, payload))
            peer._inbox_cv.notify_all()

    def recv(self, src: int = None):
        with self._inbox_cv:
            while True:
                hit = next((k for k, (s, _) in enumerate(self._inbox) if src is None or s == src), None)
                if hit is not None:
                    return self._inbox.pop(hit)[1]
                self._inbox_cv.wait()

    def _exchange(self, name, group, payload, n_in, combine):
        """Post ``payload``, combine every member's (rank order), account the call."""
        import time

        t0 = time.perf_counter()
        if isinstance(payload, torch.Tensor) and payload.is_cuda:
            torch.cuda.current_stream().synchronize()   # the peers read it from their threads
        slots = group.rendezvous.exchange(group.index[self.rank], payload)
        result = combine(slots)
        dt = time.perf_counter() - t0
        n_out = int(result.numel() if isinstance(result, torch.Tensor) else np.size(result))
        self.counters.record(name, n_in, n_out, dt)
        if self.recorder is not None:
            self.recorder(name, dt)
        return result

    @staticmethod
    def _as_payload(local):
        if isinstance(local, torch.Tensor) and local.is_cuda:
            return local.to(torch.float64)
        return np.asarray(local, dtype=np.float64)

    def all_reduce(self, group: Group, local, op: str = "sum"):
        """Elementwise reduction in ascending rank order; the same result on every member."""
        if op not in ("sum", "min", "max"):
            raise ValueError(f"unknown reduction {op!r}")
        x = self._as_payload(local)
        scalar = not isinstance(x, torch.Tensor) and x.ndim == 0
        flat = x.reshape(-1) if isinstance(x, torch.Tensor) else np.atleast_1d(x)

        def combine(slots):
            if any(tuple(v.shape) != tuple(slots[0].shape) for v in slots):
                raise ValueError("all_reduce length mismatch across group")
            return _fold(slots, op)

        out = self._exchange("AllReduce", group, flat, int(np.size(flat) if not isinstance(flat, torch.Tensor)
                                                           else flat.numel()), combine)
        if isinstance(x, torch.Tensor):
            return out.reshape(x.shape)
        return float(out[0]) if scalar else out

    def all_gather(self, group: Group, local):
        """The members' arrays concatenated along the rows in ascending rank order."""
        x = self._as_payload(local)
        cat = (lambda v: torch.cat(v, dim=0)) if isinstance(x, torch.Tensor) else (lambda v: np.concatenate(v, 0))
        return self._exchange("AllGather", group, x, int(x.numel() if isinstance(x, torch.Tensor) else x.size), cat)

    def reduce_scatter(self, group: Group, local, parts: DistMap):
        """Rank-ordered sum of the members' arrays, then this member's row block."""
        x = self._as_payload(local)
        if parts.parts != group.size:
            raise ValueError(f"partition has {parts.parts} blocks for a group of {group.size}")
        if parts.total != x.shape[0]:
            raise ValueError(f"partition covers {parts.total} rows, local array has {x.shape[0]}")
        mine = parts.block(group.index[self.rank])

        def combine(slots):
            if any(tuple(v.shape) != tuple(slots[0].shape) for v in slots):
                raise ValueError("reduce_scatter length mismatch across group")
            blk = _fold(slots, "sum")[mine]
            return blk.clone() if isinstance(blk, torch.Tensor) else blk.copy()

        return self._exchange("ReduceScatter", group, x, int(x.numel() if isinstance(x, torch.Tensor) else x.size),
                              combine)


# ------------------------------------------------------------- layout ------

class RankLayout:
    """Tensor block and owned factor rows of one rank (driver.py:223-246)."""

    def __init__(self, grid: Grid, rank: int, global_dims):
        self.grid = grid
        self.rank = rank
        self.coord = grid.coord_of(rank)
        self.global_dims = tuple(int(d) for d in global_dims)
        tensor_maps = [block_partition(i, p) for i, p in zip(self.global_dims, grid.shape)]
        self.slice_rows = [m.block(c) for m, c in zip(tensor_maps, self.coord)]
        self.local_dims = tuple(s.stop - s.start for s in self.slice_rows)
        self.groups = [grid.slice_group(n, c) for n, c in enumerate(self.coord)]
        self.owned_parts = []
        self.owned_rows = []
        for n, s in enumerate(self.slice_rows):
            parts = block_partition(s.stop - s.start, self.groups[n].size)
            local = parts.block(self.groups[n].index[rank])
            self.owned_rows.append(slice(s.start + local.start, s.start + local.stop))
            self.owned_parts.append(parts)


# ------------------------------------------------------------ backends ------

class IdentityCollectives:
    """Single execution context: collectives are the identity (driver.py:186-215)."""

    parallel = False

    def __init__(self):
        self.counters = CommCounters()

    def all_reduce(self, t, op="sum", words=None):
        if op not in ("sum", "max", "min"):
            raise ValueError(f"unknown reduction {op!r}")
        return t

    def reduce_scatter(self, mode, t, parts=None):
        return t

    def all_gather(self, mode, t, parts=None, out=None):
        if out is not None and out is not t:
            out.copy_(t)
            return out
        return t


class DistCollectives:
    """torch.distributed backend, one process per GPU (NCCL) or per CPU rank (gloo).

    Ragged row blocks are zero-padded to the slice group's longest block so the
    equal-count NCCL collectives apply; the padding never enters the counters.
    """

    parallel = True

    def __init__(self, layout: RankLayout, dist_groups=None, merge_norm_gram=None):
        import torch.distributed as dist

        self.dist = dist
        self.layout = layout
        self.counters = CommCounters()
        # gloo moves host memory only: device tensors are staged through the host
        # (CPU tests and the single-GPU multi-process test); NCCL works in place.
        self.stage = dist.get_backend() == "gloo"
        # NCCL collectives run in place on the current stream, so a whole sweep
        # (kernels + collectives) can be captured as one CUDA graph; the
        # host-staged gloo path cannot.
        self.capturable = not self.stage
        # Per mode, the column norms and the Gram of the normalised factor come from ONE
        # All-Reduce of the unnormalised Gram (diag = nsq) instead of the
        # reference's two (driver.py:414,421): N fewer latency-bound collectives per sweep,
        # counted as what is sent.  Default on NCCL grids of > 1 rank; the gloo path keeps
        # the reference's schedule (and counters) unless NNCP_MERGE_NORM_GRAM=1.
        env = os.environ.get("NNCP_MERGE_NORM_GRAM")
        if merge_norm_gram is None:
            merge_norm_gram = (env == "1") if env is not None else (not self.stage and dist.get_world_size() > 1)
        self.merge_norm_gram = bool(merge_norm_gram)
        grid = layout.grid
        if dist_groups is None:
            dist_groups = make_slice_process_groups(grid)
        self.slice_pg = [dist_groups[n][c] for n, c in enumerate(layout.coord)]

    def _padded_rows(self, parts: DistMap, device):
        """Row k of the concatenated blocks -> its row in the [member][max block] padded
        layout (cached per partition and device)."""
        cache = self.__dict__.setdefault("_pad_cache", {})
        key = (tuple(parts.lengths), str(device))
        if key not in cache:
            width = parts.max_length
            idx = [k * width + i for k in range(parts.parts) for i in range(parts.lengths[k])]
            cache[key] = torch.tensor(idx, dtype=torch.int64, device=device)
        return cache[key]

    def all_reduce(self, t, op="sum", words=None):
        """``words``: the payload the reference's call carries when ``t`` also carries
        piggy-backed internal words (the status codes on beta's All-Reduce)."""
        ops = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX, "min": self.dist.ReduceOp.MIN}
        if op not in ops:
            raise ValueError(f"unknown reduction {op!r}")
        if self.stage and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=ops[op])
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=ops[op])
        w = t.numel() if words is None else int(words)
        self.counters.record("AllReduce", w, w)
        return t

    def reduce_scatter(self, mode, t, parts):
        group = self.layout.groups[mode]
        me = group.index[self.layout.rank]
        r = int(t.shape[1])
        width = parts.max_length
        if group.size == 1:
            out = t
        else:
            if all(x == width for x in parts.lengths):
                inp = t.reshape(-1)
            else:
                # ragged blocks: one scatter into the zero-padded [member][width] layout
                inp = torch.zeros((group.size * width, r), dtype=t.dtype, device=t.device)
                inp.index_copy_(0, self._padded_rows(parts, t.device), t)
                inp = inp.reshape(-1)
            if self.stage and t.is_cuda:
                out_h = torch.empty((width, r), dtype=t.dtype)
                self.dist.reduce_scatter_tensor(out_h.reshape(-1), inp.contiguous().cpu(), group=self.slice_pg[mode])
                out_full = out_h.to(t.device)
            else:
                out_full = torch.empty((width, r), dtype=t.dtype, device=t.device)
                self.dist.reduce_scatter_tensor(out_full.reshape(-1), inp.contiguous(), group=self.slice_pg[mode])
            out = out_full[: parts.lengths[me]]
        self.counters.record("ReduceScatter", t.numel(), out.numel())
        return out

    def all_gather(self, mode, t, parts, out=None):
        """Slice-group All-Gather of the owned rows; ``out`` (optional, rows x R) receives
        the gathered block directly when the group's blocks are equal (no padding,
        no concatenation copy)."""
        group = self.layout.groups[mode]
        r = int(t.shape[1])
        width = parts.max_length
        if group.size == 1:
            res = t
        elif not (self.stage and t.is_cuda) and all(x == width for x in parts.lengths):
            res = out if out is not None else torch.empty((group.size * width, r), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(res.reshape(-1), t.contiguous().reshape(-1), group=self.slice_pg[mode])
        else:
            src = torch.zeros((width, r), dtype=t.dtype, device=t.device)
            src[: t.shape[0]] = t
            if self.stage and t.is_cuda:
                full_h = torch.empty((group.size, width, r), dtype=t.dtype)
                self.dist.all_gather_into_tensor(full_h.reshape(-1), src.reshape(-1).cpu(), group=self.slice_pg[mode])
                full = full_h.to(t.device)
            else:
                full = torch.empty((group.size, width, r), dtype=t.dtype, device=t.device)
                self.dist.all_gather_into_tensor(full.reshape(-1), src.reshape(-1), group=self.slice_pg[mode])
            # drop the padding with one gather (ragged blocks)
            res = full.reshape(group.size * width, r).index_select(0, self._padded_rows(parts, full.device))
        if out is not None and res is not out:
            out.copy_(res)
            res = out
        self.counters.record("AllGather", t.numel(), res.numel())
        return res


# Collective determinism (grid.py:242-262 reduces in rank order, bitwise reproducible;
# SPEC.md:390-391): NCCL is run-to-run deterministic for a fixed algorithm / protocol /
# topology, so the grid path pins them instead of letting the tuner switch with message
# size.  Ring + LL: defined for all three collectives, lowest latency for the <= 1 MB
# messages of the NNCP sweep.  Set before the communicators are created; explicit user
# settings win.
NCCL_PINS = {"NCCL_ALGO": "Ring", "NCCL_PROTO": "LL"}


def pin_nccl_environment(debug: bool = False) -> dict:
    """setdefault NCCL_ALGO / NCCL_PROTO (and NCCL_DEBUG=INFO for the INIT subsystem when
    ``debug``: communicator-init lines that show the rank count); returns what is in effect."""
    for k, v in NCCL_PINS.items():
        os.environ.setdefault(k, v)
    if debug:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return {k: os.environ.get(k) for k in list(NCCL_PINS) + ["NCCL_DEBUG"]}


def make_slice_process_groups(grid: Grid):
    """One torch.distributed group per (mode, coordinate); every rank creates all of them."""
    import torch.distributed as dist

    groups = []
    for n in range(len(grid.shape)):
        per = []
        for c in range(grid.shape[n]):
            ranks = list(grid.slice_group(n, c).ranks)
            per.append(dist.new_group(ranks) if len(ranks) > 1 else None)
        groups.append(per)
    return groups


class _Rendezvous:
    """post -> barrier -> combine -> barrier (grid.py:96-113), with the combine
    step run between the barriers so device reads finish before slots change."""

    def __init__(self, size: int):
        self.slots = [None] * size
        self._enter = threading.Barrier(size)
        self._leave = threading.Barrier(size)

    def exchange(self, index: int, value, combine=None):
        self.slots[index] = value
        self._enter.wait()
        view = list(self.slots)
        out = combine(view) if combine is not None else view
        self._leave.wait()
        return out

    def abort(self):
        self._enter.abort()
        self._leave.abort()


class ThreadGrid:
    """Shared state of a thread-simulated grid (one rendezvous per group)."""

    def __init__(self, grid: Grid):
        self.grid = grid
        self.all_rv = _Rendezvous(grid.total)
        self.slice_rv = [[_Rendezvous(g.size) for g in per] for per in grid.slice_groups]

    def abort(self):
        self.all_rv.abort()
        for per in self.slice_rv:
            for rv in per:
                rv.abort()


class ThreadCollectives:
    """Rank-ordered collectives between worker threads on the local device(s)."""

    parallel = True

    def __init__(self, tgrid: ThreadGrid, layout: RankLayout):
        self.tgrid = tgrid
        self.layout = layout
        self.counters = CommCounters()

    @staticmethod
    def _sync():
        torch.cuda.current_stream().synchronize()

    def all_reduce(self, t, op="sum", words=None):
        if op not in ("sum", "max", "min"):
            raise ValueError(f"unknown reduction {op!r}")
        self._sync()

        def combine(slots):
            out = slots[0].clone()
            for s in slots[1:]:  # ascending rank order (grid.py:250-262)
                if op == "sum":
                    out += s
                elif op == "max":
                    torch.maximum(out, s, out=out)
                else:
                    torch.minimum(out, s, out=out)
            self._sync()
            return out

        out = self.tgrid.all_rv.exchange(self.layout.rank, t, combine)
        t.copy_(out)
        w = t.numel() if words is None else int(words)
        self.counters.record("AllReduce", w, w)
        return t

    def reduce_scatter(self, mode, t, parts):
        group = self.layout.groups[mode]
        me = group.index[self.layout.rank]
        rv = self.tgrid.slice_rv[mode][self.layout.coord[mode]]
        self._sync()

        def combine(slots):
            blk = parts.block(me)
            out = slots[0][blk].clone()
            for s in slots[1:]:
                out += s[blk]
            self._sync()
            return out

        out = rv.exchange(me, t, combine)
        self.counters.record("ReduceScatter", t.numel(), out.numel())
        return out

    def all_gather(self, mode, t, parts, out=None):
        group = self.layout.groups[mode]
        me = group.index[self.layout.rank]
        rv = self.tgrid.slice_rv[mode][self.layout.coord[mode]]
        self._sync()

        def combine(slots):
            res = torch.cat(slots, dim=0)
            self._sync()
            return res

        res = rv.exchange(me, t, combine)
        self.counters.record("AllGather", t.numel(), res.numel())
        if out is not None:
            out.copy_(res)
            return out
        return res
