"""nncp_parallel in SPMD mode (one process per grid rank, torch.distributed) with the real kernels.

gpurun exposes one GPU, so the ranks share cuda:0 and talk over gloo (host-staged
collectives, no device-side waiting between processes); NCCL on a multi-GPU box
goes through the same DistCollectives / RankLayout / engine code with in-place
device collectives."""

import os
import socket
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1909_01149_b200 as P
        from tests.conftest import load_golden

        g = load_golden("runs.npz")
        name, grid = case[:2]
        engine = case[2] if len(case) > 2 else "auto"
        if len(case) > 3 and case[3] == "merged":
            os.environ["NNCP_MERGE_NORM_GRAM"] = "1"
        dims = tuple(int(d) for d in g[f"{name}_dims"])
        r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
        algo = str(g[f"{name}_algo"])
        x = P.DenseTensor(dims, g[f"{name}_x"])
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = P.nncp_parallel(x, P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed,
                                                 grid=grid, mttkrp_kernel=engine))
        out_q.put((rank, rep.errors, [np.asarray(f) for f in rep.model.factors],
                   [rep.counters.calls.get(c, 0) for c in ("ReduceScatter", "AllGather", "AllReduce")]))
    except Exception as exc:  # noqa: BLE001
        out_q.put((rank, repr(exc), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("hals_odd", (2, 2, 1)), ("mu4", (2, 1, 2, 1)), ("bpp3", (2, 2, 2)),
                                  ("bpp3", (2, 2, 2), "sliced"), ("mu4", (2, 1, 2, 1), "sliced"),
                                  ("bpp3", (2, 2, 2), "auto", "merged"), ("hals_odd", (2, 2, 1), "auto", "merged")])
def test_spmd_processes_match_reference_grid_run(golden, case):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    name, grid = case[:2]
    world = int(np.prod(grid))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, case, q)) for k in range(world)]
    for p in procs:
        p.start()
    results = dict((item[0], item[1:]) for item in (q.get(timeout=900) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
    g = golden("runs.npz")
    tag = f"grid_{name}_" + "x".join(map(str, grid))
    for rank in range(world):
        errors, factors, calls = results[rank]
        assert not isinstance(errors, str), errors
        assert np.max(np.abs(np.array(errors) - g[f"{tag}_errors"])) <= 1e-9
        for n, f in enumerate(factors):
            assert np.max(np.abs(f - g[f"{tag}_f{n}"])) <= 1e-6
        # merged counters: the reference's per-worker collective calls summed over workers
        want = list(g[f"{tag}_calls"])
        if len(case) > 3 and case[3] == "merged":
            # one All-Reduce per mode and sweep instead of two (norms + Gram), every worker
            r, iters, _ = (int(v) for v in g[f"{name}_meta"])
            want[2] -= world * len(grid) * iters
            if str(g[f"{name}_algo"]) == "hals":   # the reference's discarded per-column hook calls
                want[2] -= world * len(grid) * r * iters
            assert calls == want, (calls, want)
        elif str(g[f"{name}_algo"]) != "hals":
            assert calls == want


def _nccl_graph_worker(port, out_q):
    """World-size-1 NCCL job: nncp_parallel on the trivial grid goes through
    DistCollectives (in-place NCCL all-reduces on the current stream), so the
    sweep graph captures the collectives together with the kernels."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_1909_01149_b200 as P
        from tests.conftest import load_golden

        g = load_golden("runs.npz")
        res = {}
        for name in ("hals_odd", "bpp3", "mu4"):
            dims = tuple(int(d) for d in g[f"{name}_dims"])
            r, iters, iseed = (int(v) for v in g[f"{name}_meta"])
            algo = str(g[f"{name}_algo"])
            x = P.DenseTensor(dims, g[f"{name}_x"])
            out = {}
            for mode in (None, False):
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    warnings.filterwarnings("error", message="CUDA graph capture failed")
                    cfg = P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed,
                                      grid=(1,) * len(dims), cuda_graph=mode)
                    rep = P.nncp_parallel(x, cfg)
                out[mode] = (rep.errors, [np.asarray(f) for f in rep.model.factors], rep.counters.snapshot())
            seq = P.nncp_sequential(x, P.RunConfig(rank=r, algorithm=algo, max_iters=iters, tol=0.0, seed=iseed))
            res[name] = (out, seq.errors, [np.asarray(f) for f in seq.model.factors])
        out_q.put(res)
    except Exception as exc:  # noqa: BLE001
        import traceback

        out_q.put(repr(exc) + traceback.format_exc())
    finally:
        dist.destroy_process_group()


def test_nccl_sweep_graph_capture_matches_eager_and_sequential():
    """The NCCL grid path captured as a CUDA graph: bitwise the eager NCCL run and
    the sequential run, with the collective counters of the eager run."""
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_graph_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=900)
    p.join(timeout=120)
    assert not isinstance(res, str), res
    for name, (out, seq_err, seq_f) in res.items():
        (eg, fg, cg), (ee, fe, ce) = out[None], out[False]
        assert eg == ee == seq_err, name
        for a, b, c in zip(fg, fe, seq_f):
            assert np.array_equal(a, b) and np.array_equal(a, c), name
        assert cg == ce, (name, cg, ce)
        assert cg["calls"]["AllReduce"] > 0


def _fault_worker(rank, world, port, out_q):
    """Rank 1's mode-2 update in iteration 2 reports BPP cycling (row 7): every rank must
    raise the same wrapped error in the same iteration, none may block in a collective."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["NNCP_TEST_INJECT_FAULT"] = "1:2:1:1:7"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1909_01149_b200 as P
        from tests.conftest import load_golden

        g = load_golden("runs.npz")
        dims = tuple(int(d) for d in g["bpp3_dims"])
        x = P.DenseTensor(dims, g["bpp3_x"])
        try:
            P.nncp_parallel(x, P.RunConfig(rank=4, algorithm="bpp", max_iters=5, tol=0.0, grid=(2, 1, 1)))
            out_q.put((rank, "no error"))
        except RuntimeError as exc:
            cause = exc.__cause__
            out_q.put((rank, (str(exc), type(cause).__name__, getattr(cause, "column", None))))
    except Exception as exc:  # noqa: BLE001
        out_q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_spmd_failure_on_one_rank_raises_everywhere():
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fault_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))      # a hang would time out here
    for p in procs:
        p.join(timeout=120)
    for k in range(2):
        assert out[k] == ("NNLS update failed at iteration 2, mode 2", "BppCyclingError", 7), (k, out[k])


def test_thread_grid_failure_on_one_worker_raises(golden, monkeypatch):
    """The same hand-off in the thread-simulated grid (rank-ordered device reductions)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1909_01149_b200 as P
    from paper_1909_01149_b200.updaters import BppCyclingError

    monkeypatch.setenv("NNCP_TEST_INJECT_FAULT", "3:1:2:1:4")
    g = golden("runs.npz")
    dims = tuple(int(d) for d in g["bpp3_dims"])
    with pytest.raises(RuntimeError, match="iteration 1, mode 3") as info:
        P.nncp_parallel(P.DenseTensor(dims, g["bpp3_x"]),
                        P.RunConfig(rank=4, algorithm="bpp", max_iters=3, tol=0.0, grid=(2, 2, 1)))
    assert isinstance(info.value.__cause__, BppCyclingError) and info.value.__cause__.column == 4
