"""B200-native dense NNCP hot path (PLANC, arXiv 1909.01149), drop-in for the
reference package `nncp`'s alternating-update path.

Public names mirror `nncp/__init__.py:9-63` for the in-scope surface:
dimension-tree MTTKRP, Gram/Hadamard, MU / HALS / ANLS-BPP updates, the
Gram-trick error and the N-d grid.  All numerics run in libnncp_b200.so
(sm_100a); there is no CPU fallback.
"""

from .dimtree import (DimTreeContext, DimTreePlan, TempTensor, choose_balanced_split,  # noqa: F401
                      choose_split_mode, multi_ttv, partial_mttkrp)
from .driver import (ALGORITHMS, CATEGORIES, IN_SCOPE_ALGORITHMS, RunConfig, RunReport, init_factor,  # noqa: F401
                     nncp_parallel, nncp_sequential, record_category, relative_error, run_local)
from .grid import CommCounters, DistMap, Grid, Worker, block_partition  # noqa: F401
from .tensor_ops import (DenseTensor, FactorSet, gram, hadamard_grams_excluding, khatri_rao,  # noqa: F401
                         matrix_inner_product, naive_mttkrp, norm_squared, normalize_columns, reconstruct)
from .updaters import (BppCyclingError, UpdateInputs, UpdaterState, admm_update, bpp_update,  # noqa: F401
                       hals_update, mu_update, nesterov_outer_accelerate, nesterov_update, ucp_update)
from .synth import synthetic_tensor, truth_factors  # noqa: F401
from .tensor_io import (SyntheticSpec, TensorFileError, generate_synthetic, read_matrix, read_tensor,  # noqa: F401
                        write_matrix, write_tensor)

__version__ = "0.1.0"
