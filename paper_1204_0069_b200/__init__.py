"""B200-native hot path of cooperative conjugate gradient (cCG, arXiv 1204.0069).

Drop-in for the reference's ``ccg_solve`` (coopcg/solvers.hpp:329-333): the
per-iteration block CG update -- Q = A.D with the Gram reductions, the p x p
step solves for alpha and beta, and the X/R/D updates -- runs as hand-written
sm_100a CUDA kernels behind the C ABI in ``include/coopcg_gpu.h``.
"""
from .solver import (  # noqa: F401
    CudaError,
    DimensionError,
    Error,
    GpuContext,
    GpuOptions,
    IterationRecord,
    NumericalBreakdownError,
    SingularMatrixError,
    SolveOptions,
    SolveTrace,
    SpdViolationError,
    TerminalStatus,
    ccg_solve,
    cg_solve,
    steepest_descent_solve,
    gen_householder_factors,
    gen_random_spd_spectrum,
    gen_reference_rhs_starts,
    gen_rhs,
    gen_starts,
    iteration_mults,
    library_version,
    nccl_unique_id,
    row_split,
)
from .configs import CONFIGS, make_problem_on_device, make_reference_problem_on_device  # noqa: F401
