"""One BPP update of c3blk8-like shape (order-4 Grams, 256 rows, R=32) through the
C-ABI, for ncu: python tools/bpp_profile.py [rows] [rank] [reps]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1909_01149_b200 import _lib

    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    r = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    order = 4
    rng = np.random.default_rng(0)
    hs = [rng.random((128, r)) for _ in range(order)]
    hs = [h / np.linalg.norm(h, axis=0) for h in hs]
    g = np.stack([h.T @ h for h in hs])
    s = np.prod(g[:3], axis=0)
    xtrue = np.maximum(rng.standard_normal((rows, r)) + 0.8, 0.0)    # a few zeros per row
    slack = np.where(xtrue > 0.0, 0.0, rng.random((rows, r)) + 0.1)    # strictly complementary duals
    m = xtrue @ s - slack
    lib = _lib.load()
    dg, dm = torch.as_tensor(g, device="cuda"), torch.as_tensor(m, device="cuda")
    cur = torch.zeros_like(dm)
    out = torch.empty_like(dm)
    status = torch.zeros(_lib.STATUS_WORDS, dtype=torch.int32, device="cuda")
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    sets = torch.zeros(rows, dtype=torch.int64, device="cuda")
    st = _lib.stream_handle()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for k in range(reps):
        ev[2 * k].record()
        _lib.check(lib.nncp_status_reset(_lib.ptr(status), st))
        _lib.check(lib.nncp_update_ex(3, _lib.ptr(dg), order, order - 1, r, _lib.ptr(dm), _lib.ptr(cur), None, rows,
                                      _lib.ptr(out), None, None, _lib.ptr(status), 1e-16,
                                      _lib.ptr(sets) if k % 2 else None, 0,
                                      _lib.vp(ws.data_ptr()), ws.numel(), st))
        ev[2 * k + 1].record()
    torch.cuda.synchronize()
    print("per-call us:", [round(1e3 * ev[2 * k].elapsed_time(ev[2 * k + 1]), 1) for k in range(reps)])
    err = np.max(np.abs(out.cpu().numpy() - xtrue))
    print(f"bpp rows={rows} R={r}: max |x - x_true| = {err:.2e}, status {status.cpu().tolist()}")


if __name__ == "__main__":
    main()
