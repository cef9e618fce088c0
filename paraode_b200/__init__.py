"""paraode_b200 — B200-native (sm_100a) ParaIEKS: the time-parallel
probabilistic ODE solver of arXiv 2310.01145, behind the reference's solver
API (proj/include/paraode) and the C ABI include/paraode_b200.h."""
from .api import (Context, CudaError, DimensionError, FilteringElements, IeksConfig,  # noqa: F401
                  InitialValueProblem, InvalidInputError, IwpPrior, LinearGaussianChain,
                  LinearizationError, RtsResult, ScanError, SingularFactorError, SmoothingElements,
                  SolverError, SolverReport, UnsupportedError, affine, associative_scan_filtering,
                  associative_scan_smoothing, combine_filtering, combine_smoothing, default_context,
                  fitzhugh_nagumo, logistic, make_filtering_elements, make_smoothing_elements, pole,
                  eks_solve, para_ieks, para_ieks_batch, para_ieks_fused_batch, para_ieks_sharded, para_rts, pleiades, problem_by_name, rigid_body,
                  shard_range, ShardReport, torch_allgather, torch_nccl_bind, nccl_unique_id, uniform_grid, van_der_pol)
from ._abi import LIB_PATH, load  # noqa: F401
