"""Host cost of recording the sweep graph (Engine._capture) and of the first and later replays."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200 import driver as D  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

dims = tuple(int(d) for d in sys.argv[1].split("x"))
R = int(sys.argv[2])
x = synthetic_block(dims, truth_factors(dims, R, 1, "uniform"), 0.01, 1)
eng = D._Engine(x, dims, dims, P.RunConfig(rank=R, algorithm="hals", max_iters=100, tol=0.0),
                D.IdentityCollectives(), None, timing=False)
eng.initialise()
eng.iterate(1)
torch.cuda.synchronize()
t0 = time.perf_counter()
eng._capture()
torch.cuda.synchronize()
t1 = time.perf_counter()
eng.graph.replay()
torch.cuda.synchronize()
t2 = time.perf_counter()
eng.graph.replay()
torch.cuda.synchronize()
t3 = time.perf_counter()
print(f"capture {1e3 * (t1 - t0):.2f} ms, first replay {1e3 * (t2 - t1):.2f} ms, replay {1e3 * (t3 - t2):.2f} ms, "
      f"kernels in graph {eng.graph_kernels}")
