"""Independent verification helpers on the plugin API (reference oracle.py:59-95).

``windowed_argmin`` re-derives one point of a partial-exhaustion sweep with
scalar ``marginal_cost`` evaluations (so a device sweep can be checked point
by point), ``exhaustive_argmin`` scans a full value lattice, and
``monte_carlo_objective`` (montecarlo.py) estimates J by simulation with the
reference's generator and the device's per-sample costs.  The pinned closed
forms of the reference's oracle stay outside this package.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grids import window_indices
from .montecarlo import monte_carlo_objective
from .problem import NumericError, Problem

__all__ = ["OracleConfig", "exhaustive_argmin", "windowed_argmin", "monte_carlo_objective"]


@dataclass(frozen=True)
class OracleConfig:
    """Value lattice of the brute-force search (reference oracle.py:29-56)."""

    u_lo: float = -1.0
    u_hi: float = 1.0
    steps: int = 2001
    mc_samples: int = 1_000_000
    seed: int = 0

    def __post_init__(self):
        if not self.u_lo < self.u_hi:
            raise ValueError(f"oracle needs u_lo < u_hi (got {self.u_lo}, {self.u_hi})")
        if int(self.steps) != self.steps or self.steps < 2:
            raise ValueError(f"oracle.steps must be an integer of at least 2 (got {self.steps})")
        if int(self.mc_samples) != self.mc_samples or self.mc_samples < 1:
            raise ValueError(f"oracle.mc_samples must be a positive integer (got {self.mc_samples})")

    @property
    def step(self) -> float:
        return (self.u_hi - self.u_lo) / (self.steps - 1)

    def candidates(self) -> np.ndarray:
        return np.linspace(self.u_lo, self.u_hi, self.steps)


def exhaustive_argmin(problem: Problem, m: int, y: float, U, oc: OracleConfig) -> float:
    """Best response at ``y`` over the lattice; ties to the smallest value."""
    cand = oc.candidates()
    costs = problem.marginal_cost_segmented(m, cand, np.array([0, cand.size], dtype=np.int64),
                                            np.array([float(y)]), U)
    finite = np.isfinite(costs)
    if not finite.all():
        bad = int(np.flatnonzero(~finite)[0])
        raise NumericError(f"{problem.name}: non-finite marginal cost at stage {m}, u={cand[bad]}, y={y}")
    return float(cand[int(np.argmin(costs))])


def windowed_argmin(problem: Problem, m: int, y_center: float, U, radius: float) -> float:
    """The partial-exhaustion rule at one observation, with scalar evaluations."""
    g = problem.grids[m]
    vals = U.values(m)
    best_u, best_c = math.nan, math.inf
    for j in window_indices(g, y_center, radius):
        u = float(vals[j])
        if u == best_u:
            continue
        c = problem.marginal_cost(m, u, y_center, U)
        if c < best_c:
            best_c, best_u = c, u
    return best_u
