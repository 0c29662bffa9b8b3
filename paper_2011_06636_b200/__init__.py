"""B200-native Scheduled Relaxation Jacobi (SRJ) solve path (arXiv 2011.06636).

Drop-in for the reference `srj` package's solve-path API
(reference pkg/src/srj/__init__.py:9-23, hot-path subset): scheme
construction and the level ladder, the Algorithm-1 heuristic and the other
controllers, `run_cycle` / `solve`, and the problem generators of the
structured Dirichlet stencils.  The sweeps and residual norms run in
hand-written sm_100a kernels behind the C ABI in include/srj.h
(libsrj.so); there is no CPU fallback.
"""

from .chebyshev import amplification_eval, cheb_eval, cheb_roots, lambda_max, lambda_star
from .operators import (DeviceOperator, Field, StencilOperator, fill_uniform_rhs,
                        relative_residual)
from .problems import (ABSOLUTE_L2, CONFIGS, RELATIVE_L2, SOLUTION_DIFF_INF, ProblemInstance,
                       baseline_problem, config_problem, diffusion_1d_varcoef,
                       diffusion_2d_varcoef, diffusion_3d_varcoef,
                       laplace_2d_neumann, poisson_1d, poisson_2d, poisson_3d,
                       random_tridiagonal)
from .sparse import (SparseMatrix, diff_inf, matvec, relative_residual_l2, residual_l2,
                     weighted_jacobi_sweep)
from .rng import SplitMix64, derive_seed, uniform_rhs
from .schemes import (LEVEL_TABLE_M, MAX_LEVEL, ORDER_GRID_SIZE, SrjScheme,
                      generate_cjm_scheme, generate_srj_scheme, order_for_stability,
                      scheme_for_level)
from .solver import (Cjm, Controller, CycleStats, FixedM, Heuristic, Increasing, Jacobi,
                     SolveDivergedError, SolveReport, SolverState, StoppingRule,
                     average_convergence_rate, heuristic_next_level, run_cycle, solve)

__version__ = "0.1.0"
