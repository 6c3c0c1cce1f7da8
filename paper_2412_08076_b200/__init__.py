"""B200-native (sm_100a) Richardson(m) / NAG / FNS / V-cycle solve loop.

A drop-in GPU replacement for the hot path of the reference package
`richlab` (arXiv 2412.08076): repeated stencil residuals r = f - A u on
structured 2D grids, the Richardson/MOM/NAG/NAGex update with Jacobi
scaling, the fused residual-norm reduction, the DST-I spectral correction
and the V-cycle smoother/transfers.  Hand-written CUDA kernels behind a
C-ABI (include/richgpu.h, librichgpu.so); this package is the Python shim
that mirrors the reference API.
"""
from .errors import (DIVERGENCE_FACTOR, DimensionMismatch, DivergenceError, IterationState,
                     ShannonViolation, SolveReport, UnsupportedOperator, ZeroDiagonalError)
from .operator import GpuStencilOperator, JacobiScale, as_operator
from .precond import Preconditioner, TriangularPreconditioner, apply_preconditioner
from .problems import (AnisotropicProblem, HelmholtzProblem, anisotropic_stencil,
                       helmholtz_stencil)
from .richardson import (StationarySolver, inner_update, outer_sweep, solve_stationary,
                         solve_stationary_batched)
from .schedules import (WeightSchedule, chebyshev_schedule, chebyshev_semi_schedule,
                        chebyshev_semi_weights, chebyshev_weights, leja_order,
                        stencil_symbol_bounds)
# the reference's top-level names for the rest of the path (richlab/__init__.py:4-31)
from .fns import (SpectralCorrection, dst2, dst2_inv, fns_lite_step, sine_basis_eigenvalues,
                  sine_mode, solve_fns, solve_fns_batched)
from .multigrid import (build_hierarchy, prolong, prolongation_matrix, restrict,
                        restriction_matrix, v_cycle)
from .fgmres import FgmresConfig, fgmres
from .spectral import SpectralBounds, estimate_lambda_max, estimate_lambda_min

__version__ = "0.1.0"
__all__ = [n for n in dir() if not n.startswith("_")]
