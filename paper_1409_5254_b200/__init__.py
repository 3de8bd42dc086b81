"""B200-native time-multigrid slab sweep (arXiv 1409.5254), drop-in for the
reference package ``timemg``'s solver API.  Host assembly mirrors the
reference bit for bit; every cycle, sweep, norm and coarse solve runs in
hand-written sm_100a CUDA kernels behind the C ABI in include/timemg_b200.h.
"""

from .assembly import (ALPHA_MIN, BasisSpec, BlockLU, GlobalSystem, LocalOperators, RadauRule,
                       alpha, apply_global, assemble_local, basis_derivatives, basis_values,
                       build_transfers, optimal_omega, radau_rule, resolve_damping, rhs_moments,
                       stability_function)
from .hierarchy import CycleConfig, Level, SolveStats, TimeHierarchy
from .solver import (DevicePlan, block_jacobi_sweep, forward_solve, measure_convergence_factor,
                     measure_convergence_factors, random_initial_guess, solve, solve_batched,
                     solve_batched_stream,
                     two_grid_cycle, v_cycle)
from .rhs import rhs_moments_device, rhs_moments_samples, rhs_moments_sines

__version__ = "0.1.0"
