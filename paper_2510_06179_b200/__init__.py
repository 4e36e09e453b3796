"""B200-native DiffMPC hot path: batched SQP solve + IFT adjoint gradient of
parametric OCPs through a block-tridiagonal Schur complement solved by a
stair-preconditioned PCG (arXiv 2510.06179), as sm_100a CUDA kernels behind
the C ABI of include/docp_cuda.h. See DESIGN.md."""
from .api import (  # noqa: F401
    Batch, BackwardResult, BatchItem, BreakdownError, CudaError, DimensionError, DivergenceError, Error,
    EvaluationError, NumericalError, PcgConfig, RolloutTruncation, SolveResult, SqpConfig, WarmStartCache,
    affine_quadratic, attitude, drift, drift_thetas,
    backward_vjp, backward_vjp_batch, batch_solve, cartpole, describe, flat_offset, generate_affine_quadratic,
    generate_cartpole_x0, generate_drift_sequence, generate_uniform, kernel_launches,
    one_shot_config, pcg_invocations, sizes, sqp_solve, sqp_solve_batch, theta_size,
)
from . import _lib  # noqa: F401
