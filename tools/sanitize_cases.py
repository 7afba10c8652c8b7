"""Small launches of the hot kernels for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py sliced

Cases (each one launch per kernel of interest, results checked against the oracle so a
sanitizer-perturbed run that computes garbage is visible too):
  sliced  -- nncp_slice_tensor + sliced_gemm_kernel left (2 contraction chunks, K > 16384)
             and right (split-K groups), R = 32
  fp64    -- mttkrp_left_tma / mttkrp_right_tma (TMA + DMMA, KRP rows built in smem)
  bpp     -- bpp_kernel (warp-per-row active-set LU), plus MU / HALS update_rows_kernel
  ttv     -- trailing / leading multi-TTV kernels
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main(case):
    import torch

    import paper_1909_01149_b200 as P
    from oracle import nncp_oracle as O
    from paper_1909_01149_b200.dimtree import SlicedTensor

    rng = np.random.default_rng(0)
    if case in ("sliced", "fp64"):
        dims, r = ((64, 32, 16500), 32) if case == "sliced" else ((96, 80, 700), 16)
        x = rng.random(int(np.prod(dims)))
        hs = [rng.random((d, r)) for d in dims]
        plan = P.DimTreePlan.create(dims, r)
        xd = P.DenseTensor(dims, x).to_device()
        sl = SlicedTensor(xd, dims, plan.split, 6) if case == "sliced" else None
        for side, fn in (("left", O.partial_left), ("right", O.partial_right)):
            got = P.partial_mttkrp(xd, hs, side, plan, sliced=sl).data.cpu().numpy()
            err = rel(got, fn(x, dims, plan.split, hs))
            print(f"{case} {side}: rel err {err:.2e}")
            assert err <= 1e-12
    elif case == "bpp":
        r, rows = 16, 96
        a = rng.random((64, r))
        s = a.T @ a + 1e-3 * np.eye(r)
        m = rng.standard_normal((rows, r))
        cur = rng.random((rows, r))
        for algo, fn in (("bpp", O.bpp_update), ("hals", O.hals_update), ("mu", O.mu_update)):
            upd = getattr(P, f"{algo}_update")
            got = upd(P.UpdateInputs(s, np.abs(m) if algo == "mu" else m, cur))
            got = got.cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
            err = rel(got, fn(s, np.abs(m) if algo == "mu" else m, cur))
            print(f"{algo}: rel err {err:.2e}")
            assert err <= 1e-12
    elif case == "ttv":
        dims, r = (40, 30, 20), 8
        t = rng.random(dims[0] * dims[1] * r)
        c1, c0 = rng.random((dims[1], r)), rng.random((dims[0], r))
        temp = P.TempTensor(dims[:2], r, torch.as_tensor(t, device="cuda"))
        got = P.multi_ttv(temp, c1, "trailing").data.cpu().numpy()
        err = rel(got, O.ttv_trailing(t, dims[0], r, c1))
        print(f"ttv trailing: rel err {err:.2e}")
        got = P.multi_ttv(temp, c0, "leading").data.cpu().numpy()
        err2 = rel(got, O.ttv_leading(t, dims[0], r, c0))
        print(f"ttv leading: rel err {err2:.2e}")
        assert max(err, err2) <= 1e-12
    else:
        raise SystemExit(f"unknown case {case!r}")
    torch.cuda.synchronize()
    print(f"{case}: ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "sliced")
