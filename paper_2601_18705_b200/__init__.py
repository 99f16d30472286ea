"""B200-native SN-like DLR hot path.

Re-exports the names of the reference package's public surface that lie on
the hot path (``greytrt/__init__.py:3-57``), with the same call signatures
and exceptions, plus the step API itself.  Arrays are device (CUDA fp64)
tensors; ``compat.step_collocation`` is the numpy-in / numpy-out drop-in for
callers holding the reference's own objects.  The driver / CLI / presets /
material maps of the reference are out of scope.
"""

from .angular import AngularBasis, QuadratureSet, build_quadrature, orthonormalize
from .dlr_sn import CollocationStepInfo, step_collocation
from .errors import (
    CgError,
    ConfigurationError,
    ContractViolation,
    InterpolationError,
    InterpolationTieError,
    IterationLimitError,
    SolverError,
)
from .lowrank import DlrState, deim_select, evaluate_rows, solve_row_system
from .mesh import Grid, build_grid
from .physics import LinearizedStep, PhysicsConstants, linearize, planck, update_temperature
from .transport import assemble_operators, source_iteration, sweep_solve

__all__ = [
    "AngularBasis", "QuadratureSet", "build_quadrature", "orthonormalize",
    "CollocationStepInfo", "step_collocation",
    "CgError", "ConfigurationError", "ContractViolation", "InterpolationError",
    "InterpolationTieError", "IterationLimitError", "SolverError",
    "DlrState", "deim_select", "evaluate_rows", "solve_row_system",
    "Grid", "build_grid",
    "LinearizedStep", "PhysicsConstants", "linearize", "planck", "update_temperature",
    "assemble_operators", "source_iteration", "sweep_solve",
]

__version__ = "0.2.0"
