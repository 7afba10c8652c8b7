import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1909_01149_b200 as P
from oracle import nncp_oracle as O
dims, r = (256, 256, 304), 8
rng = np.random.default_rng(7)
x = rng.random(int(np.prod(dims)))
hs = [rng.random((d, r)) for d in dims]
plan = P.DimTreePlan.create(dims, r)
xd = P.DenseTensor(dims, x).to_device()
hd = [torch.from_numpy(h).cuda() for h in hs]
want = O.partial_left(x, dims, plan.split, hs)
outs = []
for k in range(20):
    got = P.partial_mttkrp(xd, hd, "left", plan).data.cpu().numpy()
    outs.append(got)
idx = [np.nonzero(o != want)[0] for o in outs]
np.savez_compressed("gpurun_out/debug_left.npz", **{f"i{k}": i for k, i in enumerate(idx)},
                    **{f"v{k}": o[i] for k, (o, i) in enumerate(zip(outs, idx))})
print("saved", [int(i.size) for i in idx])
