"""Repeat partial MTTKRPs and check bitwise reproducibility + oracle parity."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_01149_b200 as P  # noqa: E402
from oracle import nncp_oracle as O  # noqa: E402

shapes = [((256, 256, 300), 8), ((256, 256, 300), 32), ((256, 256, 304), 8), ((128, 128, 300), 8),
          ((512, 512, 64), 16), ((512, 512, 512), 16), ((128, 96, 80), 32), ((4096, 64, 32), 20)]
if len(sys.argv) > 2:
    sides_only = sys.argv[2]
else:
    sides_only = "left,right"
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for dims, r in shapes:
    rng = np.random.default_rng(sum(dims) + r)
    x = rng.random(int(np.prod(dims)))
    hs = [rng.random((d, r)) for d in dims]
    plan = P.DimTreePlan.create(dims, r)
    xd = P.DenseTensor(dims, x).to_device()
    hd = [torch.from_numpy(h).cuda() for h in hs]
    for side, fn in [(sd, f) for sd, f in (("left", O.partial_left), ("right", O.partial_right)) if sd in sides_only]:
        want = fn(x, dims, plan.split, hs)
        first = None
        bad = 0
        worst = 0.0
        for k in range(reps):
            got = P.partial_mttkrp(xd, hd, side, plan).data.cpu().numpy()
            err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
            worst = max(worst, err)
            if first is None:
                first = got
            elif not np.array_equal(first, got):
                bad += 1
                if bad <= 3:
                    diff = np.nonzero(first != got)[0]
                    print("  mismatch rep", k, "n", diff.size, "first idx", diff[:8], flush=True)
        print(dims, r, side, "nondeterministic reps:", bad, "worst rel err %.3e" % worst, flush=True)
