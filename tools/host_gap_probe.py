"""How much of a timed ALS iteration is host turnaround: back-to-back sweep-graph replays
(no per-iteration eps read) vs Engine.iterate (sync + eps/status read every iteration)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import driver as D  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

for spec in sys.argv[1:]:
    d, R, algo = spec.split(":")
    dims = tuple(int(v) for v in d.split("x"))
    R = int(R)
    fs = truth_factors(dims, R, 1, "uniform")
    x = synthetic_block(dims, fs, 0.01, 1)
    cfg = P.RunConfig(rank=R, algorithm=algo, max_iters=1000, tol=0.0)
    eng = D._Engine(x, dims, dims, cfg, D.IdentityCollectives(), None, timing=False)
    eng.initialise()
    eng.iterate(4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record()
    eng.iterate(K)
    e1.record()
    torch.cuda.synchronize()
    t_it = e0.elapsed_time(e1) / K
    e0.record()
    for _ in range(K):
        eng.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    t_gr = e0.elapsed_time(e1) / K
    print(f"{spec:24s} iterate {t_it:8.4f} ms   graph back-to-back {t_gr:8.4f} ms   gap {1e3 * (t_it - t_gr):7.1f} us",
          flush=True)
    del eng, x
    torch.cuda.empty_cache()
