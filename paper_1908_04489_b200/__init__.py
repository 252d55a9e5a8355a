"""paper_1908_04489_b200 -- B200-native marginal-cost minimisation for the
arXiv 1908.04489 UCP solver (Witsenhausen counterexample).

Mirrors the reference package ``ucpsolve``'s public API for the hot path
(problem plugin, solver loop, controllers, kernels), with every per-point
evaluation running in hand-written sm_100a CUDA kernels (libucp_b200.so,
C ABI in include/ucp_b200.h).  See DESIGN.md.
"""
from . import _lib, kernels
from .distributed import LOCAL, Sharding, from_process_group
from .grids import (
    ControllerSet,
    Grid,
    SampledController,
    eval_controller,
    eval_controller_many,
    init_identity,
    make_grid,
    nearest_index,
    nearest_indices,
    node_window_bounds,
    window_bounds,
    window_indices,
)
from .numerics import Density, Gaussian, Uniform, fd_first, fd_second, pdf, trapezoid
from .problem import NumericError, Problem
from .solver import (
    RoundReport,
    SolveResult,
    SolverConfig,
    adaptive_allocation,
    local_update_phase,
    newton_or_gradient_step,
    partial_exhaustion_phase,
    run_block,
    solve,
    solve_many,
)
from .verify import (OracleConfig, exhaustive_argmin, exhaustive_argmin_many, monte_carlo_objective, windowed_argmin,
                     windowed_argmin_many)
from .montecarlo import device_monte_carlo_objective
from .batch import solve_batch
from .comm import CommSharding, NcclComm
from .witsenhausen import Witsenhausen
from .config5 import Inventory, ZeroDelay

BACKEND = "b200"
__version__ = "0.1.0"

REGISTRY = {Witsenhausen.name: Witsenhausen, ZeroDelay.name: ZeroDelay, Inventory.name: Inventory}


def make_problem(name: str, params: dict | None = None, grids=None):
    """Instantiate a registered problem (reference problems/__init__.py:20-28)."""
    try:
        cls = REGISTRY[name]
    except KeyError:
        raise ValueError(f"problem must be one of {sorted(REGISTRY)} (got {name!r})") from None
    return cls(**(params or {}), grids=grids)


def max_workers() -> int:
    return 1


def set_workers(n: int) -> int:
    if n < 1:
        raise ValueError(f"workers must be at least 1 (got {n})")
    return 1


__all__ = [
    "BACKEND", "ControllerSet", "Density", "Gaussian", "Grid", "LOCAL", "NumericError", "Problem",
    "REGISTRY", "RoundReport", "SampledController", "Sharding", "SolveResult", "SolverConfig", "Uniform",
    "Witsenhausen", "ZeroDelay", "Inventory", "adaptive_allocation", "eval_controller", "eval_controller_many", "from_process_group",
    "init_identity", "local_update_phase", "fd_first", "fd_second", "OracleConfig", "exhaustive_argmin", "monte_carlo_objective", "device_monte_carlo_objective", "solve_batch", "NcclComm", "CommSharding",
    "windowed_argmin", "windowed_argmin_many", "exhaustive_argmin_many", "make_grid", "make_problem", "max_workers", "nearest_index",
    "nearest_indices", "newton_or_gradient_step", "node_window_bounds", "partial_exhaustion_phase", "pdf",
    "run_block", "set_workers", "solve", "solve_many", "trapezoid", "window_bounds", "window_indices", "__version__",
]
