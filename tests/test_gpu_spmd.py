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
                                  ("bpp3", (2, 2, 2), "sliced"), ("mu4", (2, 1, 2, 1), "sliced")])
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
        if str(g[f"{name}_algo"]) != "hals":
            assert calls == list(g[f"{tag}_calls"])
