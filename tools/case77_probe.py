import sys, numpy as np, warnings
warnings.simplefilter("ignore")
sys.path.insert(0, ".")
from oracle import nncp_oracle as O
import paper_1909_01149_b200 as P
for strict in (False, True):
  for seed in range(3):
    rng=np.random.default_rng(seed)
    dims=(4,5,4,6); rank=40
    hs=[rng.random((d,rank)) for d in dims]
    x=O.khatri_rao(hs)@np.ones(rank); x=x+0.05*np.sqrt(np.mean(x*x))*np.abs(rng.standard_normal(x.size))
    X=P.DenseTensor(dims,x)
    cfg=dict(rank=rank, algorithm="hals", max_iters=4, tol=0.0, seed=seed, strict_split=strict, mttkrp_kernel="fp64")
    s=P.nncp_sequential(X, P.RunConfig(**cfg)); p=P.nncp_parallel(X, P.RunConfig(grid=(3,1,2,3), **cfg))
    print(strict, seed, "seq ", np.array(s.errors)); print(strict, seed, "grid", np.array(p.errors))
