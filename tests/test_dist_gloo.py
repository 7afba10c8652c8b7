"""World-size-2 (and 4) torch.distributed/gloo tests of the N>1 data path.

Each process builds its RankLayout, computes its LOCAL partial MTTKRP with the
CPU oracle (test-side checker), and the product's DistCollectives perform the
Reduce-Scatter / All-Gather / All-Reduce of the inner iteration.  The result
must equal the global MTTKRP's owned rows, and the word counters must match
the reference's cost model (test_driver.py:252-289)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import nncp_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, grid, dims, r, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1909_01149_b200.grid import DistCollectives, Grid, RankLayout

        g = Grid(grid)
        lay = RankLayout(g, rank, dims)
        coll = DistCollectives(lay)
        rng = np.random.default_rng(5)
        x = rng.random(int(np.prod(dims)))
        hs = [rng.random((d, r)) for d in dims]
        xa = x.reshape(dims, order="F")
        xl = np.ascontiguousarray(xa[tuple(lay.slice_rows)]).ravel(order="F")
        res = {}
        for n in range(len(dims)):
            local_hs = [h[s] for h, s in zip(hs, lay.slice_rows)]
            mloc = O.naive_mttkrp(xl, lay.local_dims, local_hs, n)
            owned = coll.reduce_scatter(n, torch.from_numpy(np.ascontiguousarray(mloc)), lay.owned_parts[n])
            glob = O.naive_mttkrp(x, dims, hs, n)
            res[f"rs{n}"] = float(np.max(np.abs(owned.numpy() - glob[lay.owned_rows[n]])))
            gathered = coll.all_gather(n, torch.from_numpy(np.ascontiguousarray(hs[n][lay.owned_rows[n]])),
                                       lay.owned_parts[n])
            res[f"ag{n}"] = float(np.max(np.abs(gathered.numpy() - hs[n][lay.slice_rows[n]]))) \
                if gathered.numel() else 0.0
            # into a caller buffer (the engine gathers straight into its slice rows)
            dst = torch.full((lay.local_dims[n], r), np.nan, dtype=torch.float64)
            back = coll.all_gather(n, torch.from_numpy(np.ascontiguousarray(hs[n][lay.owned_rows[n]])),
                                   lay.owned_parts[n], out=dst)
            res[f"ago{n}"] = (back is dst, bool(np.array_equal(dst.numpy(), hs[n][lay.slice_rows[n]])))
        t = torch.full((r * r + r,), float(rank + 1), dtype=torch.float64)
        coll.all_reduce(t)
        res["ar"] = float(t[0])
        res["counters"] = (coll.counters.calls, coll.counters.words_in, coll.counters.words_out)
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(grid, dims, r):
    world = int(np.prod(grid))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, grid, dims, r, q)) for k in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("grid,dims,r", [((2, 1, 1), (7, 5, 6), 2), ((1, 2, 1), (8, 8, 8), 3),
                                         ((2, 2, 1), (7, 5, 6), 2)])
def test_gloo_collectives_reproduce_global_mttkrp(grid, dims, r):
    out = _run(grid, dims, r)
    world = int(np.prod(grid))
    for k in range(world):
        res = out[k]
        for n in range(len(dims)):
            assert res[f"rs{n}"] <= 1e-12, (k, n)
            assert res[f"ag{n}"] == 0.0, (k, n)
            assert res[f"ago{n}"] == (True, True), (k, n)
        assert res["ar"] == sum(range(1, world + 1))
        calls, win, wout = res["counters"]
        assert calls["ReduceScatter"] == len(dims) and calls["AllGather"] == 2 * len(dims)
        assert calls["AllReduce"] == 1 and win["AllReduce"] == r * r + r
        # reference cost model: Reduce-Scatter input = I_n/P_n rows x R (test_acceptance.py:243-252)
        from paper_1909_01149_b200.grid import Grid, RankLayout

        lay = RankLayout(Grid(grid), k, dims)
        assert win["ReduceScatter"] == sum(d * r for d in lay.local_dims)
        assert wout["AllGather"] == 2 * sum(d * r for d in lay.local_dims)


def _failure_worker(rank, world, port, faults, out_q):
    """Every rank publishes its own status codes into its slot of the hand-off vector
    (what nncp_gamma_publish does on the device), one SUM All-Reduce through the
    product's DistCollectives, then the product's parser picks the error to raise."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1909_01149_b200.driver import first_failure
        from paper_1909_01149_b200.grid import DistCollectives, Grid, RankLayout
        from paper_1909_01149_b200.updaters import BppCyclingError, raise_for_code

        order = 3
        lay = RankLayout(Grid((world, 1, 1)), rank, (8, 8, 8))
        coll = DistCollectives(lay)
        vec = torch.zeros(1 + world * order, dtype=torch.float64)
        vec[0] = 0.25 * (rank + 1)                                    # this rank's beta
        for mode, kind, row in faults.get(rank, []):
            vec[1 + rank * order + mode] = float(kind * 2**32 + row)
        coll.all_reduce(vec, words=1)
        fail = first_failure(vec.tolist(), world, order)
        err = None
        if fail is not None:
            try:
                raise_for_code(fail[1], fail[2])
            except BppCyclingError as exc:
                err = ("BppCyclingError", exc.column)
            except Exception as exc:  # noqa: BLE001
                err = (type(exc).__name__, None)
        out_q.put((rank, (fail, err, float(vec[0]), coll.counters.words_in["AllReduce"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("faults,want", [
    ({1: [(2, 1, 17)]}, (2, 1, 17)),                        # one rank cycles in mode 3
    ({0: [(1, 2, 3)], 1: [(0, 1, 5), (2, 1, 9)]}, (0, 1, 5)),  # lowest mode wins, then lowest rank
    ({}, None),
])
def test_failure_handoff_same_error_on_every_rank(faults, want):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_failure_worker, args=(k, world, port, faults, q)) for k in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in range(world):
        fail, err, beta, words = out[k]
        assert fail == want, (k, fail)
        assert beta == 0.25 + 0.5                                  # beta summed as before
        assert words == 1                                          # the reference's 1-word beta All-Reduce
        if want is not None:
            assert err == (("BppCyclingError", want[2]) if want[1] == 1 else ("LinAlgError", None))
    assert out[0][:2] == out[1][:2]


def _block_worker(rank, world, port, path, grid, out_q):
    """Each rank reads only its grid block of a tensor file (nncp_parallel's per-rank load,
    driver.local_block -> tensor_io.read_tensor_block); peak RSS sampled while it reads."""
    import resource
    import threading
    import time

    import psutil

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1909_01149_b200.grid import Grid, RankLayout
        from paper_1909_01149_b200.tensor_io import read_tensor_block, read_tensor_dims

        dims = read_tensor_dims(path)
        lay = RankLayout(Grid(grid), rank, dims)
        proc = psutil.Process()
        rss0 = proc.memory_info().rss
        peak = [rss0]
        stop = threading.Event()

        def sample():
            while not stop.is_set():
                peak[0] = max(peak[0], proc.memory_info().rss)
                time.sleep(0.0005)

        t = threading.Thread(target=sample)
        t.start()
        blk = read_tensor_block(path, [s.start for s in lay.slice_rows], lay.local_dims)
        stop.set()
        t.join()
        peak[0] = max(peak[0], proc.memory_info().rss)
        dist.barrier()
        ok = bool(np.array_equal(blk, np.arange(int(np.prod(dims)), dtype=np.float64)
                                 .reshape(dims, order="F")[tuple(lay.slice_rows)].ravel(order="F")))
        out_q.put((rank, (peak[0] - rss0, blk.nbytes, ok, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss)))
    finally:
        dist.destroy_process_group()


def test_per_rank_block_load_reads_only_the_block(tmp_path):
    """Every rank's host memory grows by ~its block, never by the whole tensor
    (reference driver.py:233-236 copies only each worker's block)."""
    from paper_1909_01149_b200.tensor_io import write_tensor
    from paper_1909_01149_b200.tensor_ops import DenseTensor

    dims, grid = (256, 192, 384), (2, 2, 1)
    path = str(tmp_path / "x.nncp")
    write_tensor(path, DenseTensor(dims, np.arange(int(np.prod(dims)), dtype=np.float64)))
    full = 8 * int(np.prod(dims))
    world = int(np.prod(grid))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(k, world, port, path, grid, q)) for k in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in range(world):
        grown, block, ok, _ = out[k]
        assert ok, k
        assert block == full // world
        assert grown <= 2 * block, (k, grown, block, full)
