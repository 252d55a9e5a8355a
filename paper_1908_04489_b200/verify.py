"""Independent verification helpers on the plugin API (reference oracle.py:29-95).

The reference re-derives single points of a sweep with scalar evaluations;
here every helper has a batched form that verifies MANY observations with one
device call of ``marginal_cost_segmented`` (one segment per observation:
the device kernels evaluate all candidates of all observations at once) and
picks the argmins on the host with the reference's rules.  The reference's
single-point names remain as one-observation calls of the batched forms.

* ``exhaustive_argmin_many`` / ``exhaustive_argmin``: best response over a
  value lattice (ties to the smallest value; a non-finite cost raises
  ``NumericError`` like the reference).
* ``windowed_argmin_many`` / ``windowed_argmin``: the partial-exhaustion rule
  at arbitrary observations -- snapshot values at grid points within the
  radius, first strict minimum in window order; NaN and +inf costs never win
  (the reference's ``c < best_c`` with ``best_c`` starting at +inf), and a
  window without any cost below +inf gives NaN.
* ``monte_carlo_objective`` (montecarlo.py): J by simulation.

The pinned closed forms of the reference's oracle stay outside this package
(DESIGN.md §9).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grids import window_bounds
from .montecarlo import monte_carlo_objective
from .problem import NumericError, Problem

__all__ = ["OracleConfig", "exhaustive_argmin", "exhaustive_argmin_many", "windowed_argmin", "windowed_argmin_many",
           "monte_carlo_objective"]


@dataclass(frozen=True)
class OracleConfig:
    """Value lattice of the brute-force search and the Monte-Carlo sample
    size (reference oracle.py:29-56: same fields, defaults and messages)."""

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


def _segmented_costs(problem: Problem, m: int, cand: np.ndarray, counts: np.ndarray, ys: np.ndarray, U):
    offsets = np.zeros(counts.size + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return problem.marginal_cost_segmented(m, cand, offsets, ys, U), offsets


def exhaustive_argmin_many(problem: Problem, m: int, ys, U, oc: OracleConfig) -> np.ndarray:
    """Best response at every observation of ``ys`` over the lattice of ``oc``
    (ties to the smallest value), all (observation, value) pairs in one call."""
    ys = np.atleast_1d(np.asarray(ys, dtype=np.float64))
    lat = oc.candidates()
    costs, _ = _segmented_costs(problem, m, np.tile(lat, ys.size), np.full(ys.size, lat.size), ys, U)
    costs = costs.reshape(ys.size, lat.size)
    finite = np.isfinite(costs)
    if not finite.all():
        s, j = np.argwhere(~finite)[0]
        raise NumericError(f"{problem.name}: non-finite marginal cost at stage {m}, u={lat[j]}, y={ys[s]}")
    return lat[np.argmin(costs, axis=1)]


def exhaustive_argmin(problem: Problem, m: int, y: float, U, oc: OracleConfig) -> float:
    """Best response at ``y`` over the lattice; ties to the smallest value."""
    return float(exhaustive_argmin_many(problem, m, [float(y)], U, oc)[0])


def windowed_argmin_many(problem: Problem, m: int, ys, U, radius: float) -> np.ndarray:
    """The partial-exhaustion rule at every observation of ``ys``: candidates
    are the snapshot values at the grid points within ``radius`` (window
    order), the first strict minimum among costs below +inf wins."""
    ys = np.atleast_1d(np.asarray(ys, dtype=np.float64))
    g = problem.grids[m]
    vals = U.values(m)
    bounds = [window_bounds(g, float(y), radius) for y in ys]
    counts = np.array([hi - lo + 1 for lo, hi in bounds], dtype=np.int64)
    cand = np.concatenate([vals[lo:hi + 1] for lo, hi in bounds]) if ys.size else np.empty(0)
    costs, offsets = _segmented_costs(problem, m, cand, counts, ys, U)
    out = np.full(ys.size, np.nan)
    for s in range(ys.size):
        c = costs[offsets[s]:offsets[s + 1]]
        ok = c < np.inf  # NaN and +inf never pass the reference's `c < best_c` with best_c = +inf
        if ok.any():
            k = np.flatnonzero(ok)
            out[s] = cand[offsets[s] + k[np.argmin(c[k])]]  # np.argmin: first of equal minima
    return out


def windowed_argmin(problem: Problem, m: int, y_center: float, U, radius: float) -> float:
    """The partial-exhaustion rule at one observation."""
    return float(windowed_argmin_many(problem, m, [float(y_center)], U, radius)[0])
