"""Per-category device time of one config (CUDA events), e.g. python tools/breakdown.py c3 5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_01149_b200 as P  # noqa: E402
from paper_1909_01149_b200.synth import synthetic_block, truth_factors  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
conf = bench.CONFIGS[name]
dims, R = conf["dims"], conf["rank"]
x = synthetic_block(dims, truth_factors(dims, R, 1, conf["kind"]), conf["eta"], 1)
eng, rep = P.run_local(x, dims, dims, P.RunConfig(rank=R, algorithm=conf["algo"], max_iters=iters, tol=0.0))
rows = rep.rows[2:]
tot = {c: np.mean([r[c] for r in rows]) * 1e3 for c in P.CATEGORIES}
wall = np.mean(rep.row_wall[2:]) * 1e3
print(name, dims, R, conf["algo"], "wall ms/iter %.3f" % wall, "device categories (ms):",
      {k: round(v, 3) for k, v in tot.items() if v > 0}, "sum %.3f" % sum(tot.values()))
