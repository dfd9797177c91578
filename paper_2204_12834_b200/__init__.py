"""B200-native (sm_100a, fp64) power-series Schur solve for bundle adjustment.

Drop-in for the hot path of the reference package ``powerba`` (Power Bundle
Adjustment, arXiv 2204.12834): the same entry points and problem layout, with
every O(n_obs) operation running in the CUDA library ``lib/libpoba.so``.
"""
from .blocks import (DampedSystem, LandmarkBlockStore, Linearization, assemble,  # noqa: F401
                     assemble_from_observations, linearize, memory_account)
from .lm import (BaState, LmConfig, SolverTrace, apply_update, evaluate_cost, residual_cost,  # noqa: F401
                 run)
from .power_series import (PowerSeriesResult, apply_series_inverse, back_substitute,  # noqa: F401
                           power_series_solve, stop_criterion)
from .problem import Problem  # noqa: F401
from .solvers import (CgReport, make_schur_jacobi_preconditioner, pcg, pcg_power_series_preconditioner,  # noqa: F401
                      pcg_schur_jacobi, schur_diagonal_blocks)

from . import bal_io, clustering, solvers, spectral  # noqa: F401,E402

__version__ = "0.1.0"
