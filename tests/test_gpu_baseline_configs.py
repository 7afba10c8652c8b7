"""BASELINE.json configs c2, c3, c4 at full size against the CPU oracle.

c2 512^3 R=16 HALS 30 iterations, sequential and on the 2x2x2 grid; c4
4096x2048x256 R=20 HALS and c3 256^4 R=32 BPP, 10 iterations each: the device
run (default engine choice, the one bench.py measures) against the CPU oracle
(oracle/nncp_oracle.py, pinned to the live reference by the golden vectors)
on the same input bits.  Traces <= 1e-9 over the first 10 iterations, final
normalised factors <= 1e-6 (north_star)."""

import numpy as np
import pytest

from oracle import nncp_oracle as O

pytestmark = pytest.mark.gpu

TRACE_TOL = 1e-9
FACTOR_TOL = 1e-6

# BASELINE.json configs (bench.py CONFIGS): dims, rank, algorithm, noise eta, factor kind
CONFIGS = {
    "c2": ((512, 512, 512), 16, "hals", 0.01, "uniform"),
    "c3": ((256, 256, 256, 256), 32, "bpp", 0.01, "uniform"),
    "c4": ((4096, 2048, 256), 20, "hals", 0.05, "walk"),
}


def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return torch


def _free():
    import gc

    import torch

    gc.collect()
    torch.cuda.empty_cache()


def _config_tensor(name):
    from paper_1909_01149_b200.synth import synthetic_block, truth_factors

    dims, rank, algo, eta, kind = CONFIGS[name]
    fs = truth_factors(dims, rank, 1, kind)
    return dims, rank, algo, synthetic_block(dims, fs, eta, 1)


def _compare(rep, errors, factors, lam, tag):
    n = min(len(rep.errors), len(errors), 11)                      # init row + first 10 iterations
    trace10 = float(np.max(np.abs(np.array(rep.errors[:n]) - np.array(errors[:n]))))
    trace_all = float(np.max(np.abs(np.array(rep.errors) - np.array(errors))))
    fac = max(float(np.max(np.abs(a - b))) for a, b in zip(rep.model.factors, factors))
    print(f"{tag}: trace(first 10) {trace10:.2e}, trace(all {len(errors) - 1}) {trace_all:.2e}, "
          f"factors {fac:.2e}, eps {rep.errors[-1]:.6e}")
    assert len(rep.errors) == len(errors)
    assert trace10 <= TRACE_TOL, (tag, trace10)
    assert fac <= FACTOR_TOL, (tag, fac)
    assert np.allclose(rep.model.lam, lam, rtol=1e-6, atol=0), tag


@pytest.mark.parametrize("name,iters,grid", [("c2", 30, None), ("c2", 30, (2, 2, 2)), ("c4", 10, None),
                                             ("c3", 10, None)])
def test_baseline_config_vs_oracle(name, iters, grid):
    _cuda()
    import paper_1909_01149_b200 as P

    dims, rank, algo, xd = _config_tensor(name)
    host = xd.cpu().numpy()
    cfg = P.RunConfig(rank=rank, algorithm=algo, max_iters=iters, tol=0.0, grid=grid)
    if grid is None:
        rep = P.nncp_sequential(P.DenseTensor(dims, xd), cfg)
    else:
        rep = P.nncp_parallel(P.DenseTensor(dims, xd), cfg)
    del xd
    _free()
    # the oracle's init error goes through the tree (same quantity as the reference's einsum,
    # driver.py:362-373; the device does the same), everything else is the reference algorithm
    errors, factors, lam, split, _ = O.run_sequential(host, dims, rank, algo, iters, 0.0, 0, init_error="tree")
    _compare(rep, errors, factors, lam, f"{name} grid={grid}")
