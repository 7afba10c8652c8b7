"""Per-category device time of one ALS iteration (engine CUDA events), graph vs eager."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200.driver import _Engine  # noqa: E402
from paper_1909_01149_b200.grid import IdentityCollectives  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
R = int(sys.argv[2])
algo = sys.argv[3] if len(sys.argv) > 3 else "hals"
fs = truth_factors(dims, R, 1, "uniform")
x = synthetic_block(dims, fs, 0.01, 1)
for graph in (False, True):
    cfg = P.RunConfig(rank=R, algorithm=algo, max_iters=8, tol=0.0, seed=0, cuda_graph=graph)
    eng = _Engine(x, dims, dims, cfg, IdentityCollectives(), None, timing=True)
    eng.initialise()
    eng.iterate(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.iterate(4)
    e1.record()
    torch.cuda.synchronize()
    rows = eng.report.rows[-4:]
    cats = {k: sum(r[k] for r in rows) / 4 * 1e3 for k in rows[0]}
    print(f"graph={graph}: {e0.elapsed_time(e1) / 4:.3f} ms/iter; categories (ms): "
          + ", ".join(f"{k} {v:.3f}" for k, v in cats.items() if v > 0) + f"; sum {sum(cats.values()):.3f}", flush=True)
    del eng
    torch.cuda.empty_cache()
