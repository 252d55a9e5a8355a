"""ORACLE -- TEST INFRASTRUCTURE ONLY (parity checker, CPU baseline).

Python side of the CPU restatement of the reference's hot path.  The loops
live in ``ucp_oracle.c`` (host glibc exp/erf, OpenMP over independent
outputs); this module restates the reference's NumPy glue around them with
the same NumPy expressions, so on the same host every result is bitwise the
reference's.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline leg may import it; the product package never does.

Each function cites the reference code it restates (paths relative to
``/root/reference/pkg/src/ucpsolve``).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_dbl = ctypes.c_double

INV_SQRT_2PI = 1.0 / np.sqrt(2.0 * np.pi)  # numerics.py:22 / kernels.py:47


def build(force: bool = False) -> Path:
    """Compile ucp_oracle.c with the committed Makefile (gcc, OpenMP)."""
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "ucp_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.orc_trapezoid.restype = _dbl
        L.orc_trapezoid.argtypes = [_f64p, _i64, _dbl]
        L.orc_segmented_argmin.restype = None
        L.orc_segmented_argmin.argtypes = [_f64p, _i64p, _i64, _i64p]
        L.orc_flatten_windows.restype = _i64
        L.orc_flatten_windows.argtypes = [_f64p, _i64p, _i64p, _i64, ctypes.c_void_p, _i64p]
        L.orc_gauss_moments_grid.restype = None
        L.orc_gauss_moments_grid.argtypes = [_f64p, _i64, _f64p, _dbl, _dbl, _i64, _f64p, _f64p, _f64p]
        L.orc_gauss_moments_points.restype = None
        L.orc_gauss_moments_points.argtypes = [
            _f64p, _i64, _f64p, _f64p, _i64, _dbl, _dbl, _i64, _f64p, _f64p, _f64p]
        L.orc_wc_stage0_cost.restype = None
        L.orc_wc_stage0_cost.argtypes = [
            _f64p, _i64p, _i64, _f64p, _f64p, _f64p, _dbl, _dbl, _i64, _dbl, _f64p]
        L.orc_wc_stage1_cost.restype = None
        L.orc_wc_stage1_cost.argtypes = [
            _f64p, _i64p, _i64, _f64p, _f64p, _f64p, _i64, _dbl, _dbl, _i64, _f64p]
        L.orc_unif_moments_grid.restype = None
        L.orc_unif_moments_grid.argtypes = [_f64p, _i64, _f64p, _dbl, _dbl, _i64, _dbl, _f64p, _f64p, _f64p]
        L.orc_unif_ball_sum.restype = None
        L.orc_unif_ball_sum.argtypes = [_f64p, _i64, _f64p, _dbl, _dbl, _i64, _dbl, _f64p]
        L.orc_unif_propagate.restype = None
        L.orc_unif_propagate.argtypes = [_f64p, _f64p, _i64, _dbl, _dbl, _i64, _dbl, _f64p]
        L.orc_unif_moments_points.restype = None
        L.orc_unif_moments_points.argtypes = [_f64p, _i64, _f64p, _f64p, _f64p, _i64, _dbl, _dbl, _i64, _dbl,
                                              _f64p, _f64p, _f64p]
        L.orc_phi_cdf.restype = _dbl
        L.orc_phi_cdf.argtypes = [_dbl]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_threads.restype = None
        L.orc_set_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _c(x, dt=np.float64):
    return np.ascontiguousarray(x, dtype=dt)


# ---------------------------------------------------------------- kernels.py


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


def trapezoid_sum(samples, spacing):  # kernels.py:136-144
    s = _c(samples)
    return float(lib().orc_trapezoid(s, s.size, float(spacing)))


def segmented_argmin(costs, offsets):  # kernels.py:147-160
    c, o = _c(costs), _c(offsets, np.int64)
    out = np.empty(o.size - 1, np.int64)
    lib().orc_segmented_argmin(c, o, o.size - 1, out)
    return out


def flatten_windows(values, lo, hi):  # kernels.py:163-187 (dedup variant)
    v, lo, hi = _c(values), _c(lo, np.int64), _c(hi, np.int64)
    offsets = np.empty(lo.size + 1, np.int64)
    flat = np.empty(int(np.sum(hi - lo + 1)), np.float64)
    n = lib().orc_flatten_windows(v, lo, hi, lo.size, flat.ctypes.data, offsets)
    return flat[:n].copy(), offsets


def gauss_moments_grid(s, v, a, h, d):  # kernels.py:406-445
    s, v = _c(s), _c(v)
    t0, t1, t2 = (np.empty(s.size) for _ in range(3))
    lib().orc_gauss_moments_grid(s, s.size, v, float(a), float(h), int(d), t0, t1, t2)
    return t0, t1, t2


def gauss_moments_points(y, x, w, a, h, d):  # kernels.py:447-486
    y, x, w = _c(y), _c(x), _c(w)
    o = [np.empty(y.size) for _ in range(3)]
    lib().orc_gauss_moments_points(y, y.size, x, w, x.size, float(a), float(h), int(d), *o)
    return tuple(o)


def phi_cdf(z):  # kernels.py:398-404
    return float(lib().orc_phi_cdf(float(z)))


def unif_moments_grid(x, v, a, h, d, rad):  # kernels.py:488-525
    x, v = _c(x), _c(v)
    o = [np.empty(x.size) for _ in range(3)]
    lib().orc_unif_moments_grid(x, x.size, v, float(a), float(h), int(d), float(rad), *o)
    return tuple(o)


def unif_ball_sum(x, g, a, h, d, rad):  # kernels.py:528-555
    x, g = _c(x), _c(g)
    out = np.empty(x.size)
    lib().orc_unif_ball_sum(x, x.size, g, float(a), float(h), int(d), float(rad), out)
    return out


def unif_propagate(masses, centers, a, h, d, rad):  # kernels.py:558-577
    masses, centers = _c(masses), _c(centers)
    out = np.empty(int(d))
    lib().orc_unif_propagate(masses, centers, centers.size, float(a), float(h), int(d), float(rad), out)
    return out


def unif_moments_points(y, centers, w, vals, a, h, d, rad):  # kernels.py:580-615
    y, centers, w, vals = _c(y), _c(centers), _c(w), _c(vals)
    o = [np.empty(y.size) for _ in range(3)]
    lib().orc_unif_moments_points(y, y.size, centers, w, vals, centers.size, float(a), float(h), int(d),
                                  float(rad), *o)
    return tuple(o)


# ------------------------------------------------------ grids / numerics glue


def linspace_grid(a, b, d):  # grids.py:50 (np.linspace) and :55-56 (spacing)
    return np.linspace(float(a), float(b), int(d)), (float(b) - float(a)) / (int(d) - 1)


def gaussian_pdf(mean, std, x):  # numerics.py:49-60 (NumPy exp, not glibc)
    z = (np.asarray(x, dtype=np.float64) - mean) / std
    return np.exp(-0.5 * z * z) * (INV_SQRT_2PI / std)


def node_window_bounds(points, a, h, d, r):  # grids.py:180-195 (+ nearest_indices :141-145)
    lo = np.ceil((points - r - a) / h - 1e-9).astype(np.int64)
    hi = np.floor((points + r - a) / h + 1e-9).astype(np.int64)
    ic = np.clip(np.ceil((points - a) / h - 0.5).astype(np.int64), 0, d - 1)
    lo = np.maximum(0, np.minimum(lo, ic))
    hi = np.minimum(d - 1, np.maximum(hi, ic))
    return lo, hi


# ------------------------------------------------------------ Witsenhausen


@dataclass
class OracleWitsenhausen:
    """Restates problems/witsenhausen.py:36-79 on plain arrays.

    ``f0`` (stage-0 density at the stage-0 grid points) and ``fw0`` are the
    host NumPy values the reference computes; they may be injected so
    parity runs can share one set of host-computed constants.
    """

    k: float = 0.2
    sigma: float = 5.0
    grid0: tuple = (-25.0, 25.0, 2000)
    grid1: tuple = (-25.0, 25.0, 2000)
    f0: np.ndarray | None = None
    fw0: np.ndarray | None = None

    def __post_init__(self):
        self.y0, self.h0 = linspace_grid(*self.grid0)
        self.y1, self.h1 = linspace_grid(*self.grid1)
        self.d0, self.d1 = int(self.grid0[2]), int(self.grid1[2])
        self.a0, self.a1 = float(self.grid0[0]), float(self.grid1[0])
        if self.fw0 is None:  # witsenhausen.py:47-53
            w0 = np.full(self.d0, self.h0)
            w0[0] *= 0.5
            w0[-1] *= 0.5
            self.fw0 = w0 * gaussian_pdf(0.0, self.sigma, self.y0)
        if self.f0 is None:
            self.f0 = gaussian_pdf(0.0, self.sigma, self.y0)

    name = "witsenhausen"
    M = 2

    def grid(self, m):
        return (self.y0, self.a0, self.h0, self.d0) if m == 0 else (self.y1, self.a1, self.h1, self.d1)

    def span(self, m):
        g = self.grid0 if m == 0 else self.grid1
        return float(g[0]), float(g[1])

    def h_floor(self, m):
        return None

    def project(self, m, v):
        return v

    # witsenhausen.py:59-79.  y_centers are always stage grid points here
    # (indices `seg_idx`), whose f0 is the host-precomputed per-point value.
    def cost_segmented(self, m, u_flat, offsets, seg_idx, Us_or_u0, u1=None):
        u0, u1 = (Us_or_u0, u1) if u1 is not None else (Us_or_u0[0], Us_or_u0[1])
        u_flat, offsets = _c(u_flat), _c(offsets, np.int64)
        seg_idx = _c(seg_idx, np.int64)
        out = np.empty(u_flat.size)
        if m == 0:
            y = _c(self.y0[seg_idx])
            f0 = _c(self.f0[seg_idx])
            lib().orc_wc_stage0_cost(u_flat, offsets, offsets.size - 1, y, f0, _c(u1),
                                     self.a1, self.h1, self.d1, self.k, out)
        else:
            y = _c(self.y1[seg_idx])
            x1 = self.y0 + u0
            lib().orc_wc_stage1_cost(u_flat, offsets, offsets.size - 1, y, _c(x1), _c(self.fw0),
                                     self.d0, self.a1, self.h1, self.d1, out)
        return out

    def cost_batch(self, m, u, idx, u0, u1):  # problem.py:69-76
        u = _c(u)
        return self.cost_segmented(m, u, np.arange(u.size + 1, dtype=np.int64), idx, [u0, u1])


class OracleNumericError(RuntimeError):
    """Mirror of problem.NumericError (problem.py:25-26)."""


def nearest_idx(points, a, h, d, y):  # grids.py:141-145
    return np.clip(np.ceil((np.asarray(y, dtype=np.float64) - a) / h - 0.5).astype(np.int64), 0, d - 1)


def _trap_weights(h, d):
    w = np.full(d, h)
    w[0] *= 0.5
    w[-1] *= 0.5
    return w


class OracleZeroDelay:
    """Restates problems/zero_delay.py:36-86 (uniform channel noise U(-1, 1))."""

    name = "zero_delay"

    def __init__(self, power_weight=2.0, grid0=(-5.0, 5.0, 2000), grid1=(-6.0, 6.0, 2000), f0=None, fw0=None):
        self.pw = float(power_weight)
        self.specs = [tuple(grid0), tuple(grid1)]
        self.M = 2
        self.pts = [linspace_grid(*g)[0] for g in self.specs]
        self.hs = [linspace_grid(*g)[1] for g in self.specs]
        self.f0 = gaussian_pdf(0.0, 1.0, self.pts[0]) if f0 is None else _c(f0)
        self.fw0 = _trap_weights(self.hs[0], self.pts[0].size) * gaussian_pdf(0.0, 1.0, self.pts[0]) \
            if fw0 is None else _c(fw0)

    def grid(self, m):
        return self.pts[m], float(self.specs[m][0]), self.hs[m], int(self.specs[m][2])

    def span(self, m):
        return float(self.specs[m][0]), float(self.specs[m][1])

    def h_floor(self, m):  # zero_delay.py:56-65 (probe widened to one decoder cell)
        return self.hs[1]

    def project(self, m, v):
        return v

    def cost_segmented(self, m, u_flat, offsets, seg_idx, Us):
        counts = np.diff(offsets)
        _, a1, h1, d1 = self.grid(1)
        if m == 0:  # zero_delay.py:69-76
            y_flat = np.repeat(self.pts[0][seg_idx], counts)
            s0, s1, s2 = unif_moments_grid(u_flat, Us[1], a1, h1, d1, 1.0)
            distortion = s0 * y_flat * y_flat - 2.0 * s1 * y_flat + s2
            f0 = np.repeat(self.f0[seg_idx], counts)
            return f0 * (self.pw * u_flat * u_flat + distortion)
        a, b, c = unif_moments_points(self.pts[1][seg_idx], Us[0], self.fw0, self.pts[0], a1, h1, d1, 1.0)
        a, b, c = (np.repeat(t, counts) for t in (a, b, c))  # zero_delay.py:77-83
        return a * u_flat * u_flat - 2.0 * b * u_flat + c


class OracleInventory:
    """Restates problems/inventory.py:31-150 (M stages, uniform demand, u >= 0)."""

    name = "inventory"

    def __init__(self, stages=2, order_cost=0.1, stage_cost="piecewise_linear", holding_rate=1.0,
                 backlog_rate=1.0, grids=None):
        self.M = int(stages)
        self.oc = float(order_cost)
        self.stage_cost = stage_cost
        self.hr, self.br = float(holding_rate), float(backlog_rate)
        self.specs = [tuple(g) for g in (grids or [(-3.0, 3.0, 601)] * self.M)]
        self.pts = [linspace_grid(*g)[0] for g in self.specs]
        self.hs = [linspace_grid(*g)[1] for g in self.specs]

    def grid(self, m):
        return self.pts[m], float(self.specs[m][0]), self.hs[m], int(self.specs[m][2])

    def span(self, m):
        return float(self.specs[m][0]), float(self.specs[m][1])

    def gamma(self, x):  # inventory.py:61-69
        if self.stage_cost == "quadratic":
            return x * x
        return self.hr * np.maximum(x, 0.0) + self.br * np.maximum(-x, 0.0)

    def project(self, m, v):  # inventory.py:71-72
        return np.maximum(v, 0.0)

    def state(self, mm):  # inventory.py:74-76
        return self.grid(min(mm, self.M - 1))

    def h_floor(self, m):  # inventory.py:131-136
        return self.state(m + 1)[2]

    def downstream(self, Us):  # inventory.py:78-94
        gs = [None] * (self.M + 1)
        gs[self.M] = self.gamma(self.state(self.M)[0])
        for mm in range(self.M - 1, 0, -1):
            pts = self.pts[mm]
            _, an, hn, dn = self.state(mm + 1)
            expect = unif_ball_sum(pts + Us[mm], gs[mm + 1], an, hn, dn, 1.0)
            gs[mm] = self.gamma(pts) + (self.oc * Us[mm] + expect)
        return gs

    def forward_density(self, m, Us):  # inventory.py:96-110
        _, a0, h0, d0 = self.grid(0)
        f = unif_propagate(np.array([1.0]), np.array([0.0]), a0, h0, d0, 1.0)
        for mm in range(m):
            _, an, hn, dn = self.grid(mm + 1)
            f = unif_propagate(self.hs[mm] * f, self.pts[mm] + Us[mm], an, hn, dn, 1.0)
        return f

    def cost_segmented(self, m, u_flat, offsets, seg_idx, Us):  # inventory.py:138-150
        counts = np.diff(offsets)
        pts, a, h, d = self.grid(m)
        y_flat = np.repeat(pts[seg_idx], counts)
        f_m = self.forward_density(m, Us)
        gs = self.downstream(Us)
        _, an, hn, dn = self.state(m + 1)
        expect = unif_ball_sum(y_flat + u_flat, gs[m + 1], an, hn, dn, 1.0)
        weight = f_m[nearest_idx(pts, a, h, d, y_flat)]
        return weight * (self.oc * u_flat + expect)


@dataclass(frozen=True)
class OracleConfig:  # solver.py:47-97 (fields used on the hot path)
    iters_per_round: int = 20
    precision: float = 1e-10
    grad_step: float = 0.1
    search_radius: float | None = None
    fd_step: float = 1e-4
    curvature_min: float = 1e-9
    newton_cap: float | None = None
    max_rounds: int = 10000

    def radius(self, a, b):
        return self.search_radius if self.search_radius is not None else (b - a) / 100.0

    def cap(self, a, b):
        return self.newton_cap if self.newton_cap is not None else (b - a) / 10.0


def _bad(p, m, phase, i):
    y = p.grid(m)[0][int(i)]
    return OracleNumericError(
        f"{p.name}: non-finite marginal cost in {phase} phase at stage {m}, grid point {int(i)} (y={y!r})")


def _cost_batch(p, m, u, idx, Us):
    u = _c(u)
    return p.cost_segmented(m, u, np.arange(u.size + 1, dtype=np.int64), idx, Us)


def local_update(p, m, Us, cfg: OracleConfig, points=None):
    """solver.py:179-203 with problem.py:88-102 (and the problems' probe floors)."""
    u_all = Us[m]
    idx = np.arange(u_all.size, dtype=np.int64) if points is None else _c(points, np.int64)
    u = u_all[idx]
    with np.errstate(over="ignore"):
        h = cfg.fd_step * (1.0 + np.abs(u))
    floor = p.h_floor(m) if hasattr(p, "h_floor") else None
    if floor is not None:
        h = np.maximum(h, floor)
    up = _cost_batch(p, m, u + h, idx, Us)
    mid = _cost_batch(p, m, u, idx, Us)
    dn = _cost_batch(p, m, u - h, idx, Us)
    with np.errstate(over="ignore", invalid="ignore"):
        c1 = (up - dn) / (2.0 * h)
        c2 = (up - 2.0 * mid + dn) / (h * h)
    bad = np.flatnonzero(~(np.isfinite(c1) & np.isfinite(c2)))
    if bad.size:
        raise _bad(p, m, "local-update", idx[bad[0]])
    cap = cfg.cap(*p.span(m))
    newton = c2 > cfg.curvature_min
    quot = np.divide(c1, c2, out=np.zeros_like(c1), where=newton)
    stepped = p.project(m, np.where(newton, u - np.clip(quot, -cap, cap), u - cfg.grad_step * c1))
    cost_old = _cost_batch(p, m, u, idx, Us)
    cost_new = _cost_batch(p, m, stepped, idx, Us)
    bad = np.flatnonzero(~(np.isfinite(cost_old) & np.isfinite(cost_new)))
    if bad.size:
        raise _bad(p, m, "local-update", idx[bad[0]])
    return np.where(cost_new <= cost_old, stepped, u)


def partial_exhaustion(p, m, Us, cfg: OracleConfig, points=None):
    """solver.py:206-223 with grids.py:180-195 and kernels.py:147-187."""
    y, a, h, d = p.grid(m)
    lo, hi = node_window_bounds(y, a, h, d, cfg.radius(*p.span(m)))
    idx = np.arange(d, dtype=np.int64) if points is None else _c(points, np.int64)
    cand, offsets = flatten_windows(Us[m], lo[idx], hi[idx])
    costs = p.cost_segmented(m, cand, offsets, idx, Us)
    bad = np.flatnonzero(~np.isfinite(costs))
    if bad.size:
        seg = int(np.searchsorted(offsets, bad[0], side="right") - 1)
        raise _bad(p, m, "partial-exhaustion", idx[seg])
    return p.project(m, cand[segmented_argmin(costs, offsets)])


def objective_of(p, Us):  # problem.py:110-127
    y, a, h, d = p.grid(0)
    costs = _cost_batch(p, 0, Us[0], np.arange(d, dtype=np.int64), Us)
    bad = np.flatnonzero(~np.isfinite(costs))
    if bad.size:
        i = int(bad[0])
        raise OracleNumericError(
            f"{p.name}: non-finite objective integrand at stage 0, grid point {i} "
            f"(y={y[i]!r}, u={Us[0][i]!r})")
    return trapezoid_sum(costs, h)


def adaptive_allocation(gl, ge, n):  # solver.py:152-167
    total = gl + ge
    if total <= 0.0:
        nl = n // 2
    else:
        nl = min(max(math.floor(gl * n / total), 1), n - 1)
    return nl, n - nl


def solve_generic(p, cfg: OracleConfig | None = None, Us=None):
    """solver.py:234-290 (adaptive local/exhaustion rounds) for any oracle problem."""
    cfg = cfg or OracleConfig()
    Us = [p.grid(m)[0].copy() for m in range(p.M)] if Us is None else [_c(u).copy() for u in Us]
    Us = [p.project(m, Us[m]) for m in range(p.M)]
    n = cfg.iters_per_round
    n_local = n // 2
    current = objective_of(p, Us)
    rounds = []
    term = "max_rounds"
    for r in range(1, cfg.max_rounds + 1):
        for phase, iters in ((local_update, n_local), (partial_exhaustion, n - n_local)):
            for _ in range(iters):
                for m in range(p.M):
                    Us[m] = phase(p, m, Us, cfg)
            if phase is local_update:
                after_local = objective_of(p, Us)
        after_exh = objective_of(p, Us)
        gl, ge = abs(current - after_local), abs(after_local - after_exh)
        rounds.append((r, after_exh, gl, ge, n_local, n - n_local, after_local))
        current = after_exh
        if gl + ge <= cfg.precision:
            term = "converged"
            break
        n_local, _ = adaptive_allocation(gl, ge, n)
    return Us, current, rounds, term


# ---- Witsenhausen wrappers (two controllers passed explicitly) --------------
def local_update_phase(p, m, u0, u1, cfg: OracleConfig, points=None):
    return local_update(p, m, [u0, u1], cfg, points)


def partial_exhaustion_phase(p, m, u0, u1, cfg: OracleConfig, points=None):
    return partial_exhaustion(p, m, [u0, u1], cfg, points)


def objective(p, u0, u1):
    return objective_of(p, [u0, u1])


def solve(p, cfg: OracleConfig | None = None, u0=None, u1=None):
    Us, J, rounds, term = solve_generic(p, cfg, None if u0 is None else [u0, u1])
    return Us[0], Us[1], J, rounds, term


# ---- Monte-Carlo objective (oracle.py:98-105) -------------------------------


def simulate_cost(p, Us, draws):
    """Per-sample simulated cost from pre-drawn variates ``draws[s][i]``, the
    generator outputs in the order the reference's ``simulate_cost`` consumes
    them; the expressions are the reference's, NumPy elementwise."""
    draws = [np.asarray(d, dtype=np.float64) for d in draws]
    if p.name == "witsenhausen":  # problems/witsenhausen.py:81-89
        _, a0, h0, d0 = p.grid(0)
        _, a1, h1, d1 = p.grid(1)
        x0 = draws[0]
        u0 = np.asarray(Us[0])[nearest_idx(None, a0, h0, d0, x0)]
        x1 = x0 + u0
        w = draws[1]
        u1 = np.asarray(Us[1])[nearest_idx(None, a1, h1, d1, x1 + w)]
        x2 = x1 - u1
        return p.k * p.k * u0 * u0 + x2 * x2
    if p.name == "zero_delay":  # problems/zero_delay.py:88-94
        _, a0, h0, d0 = p.grid(0)
        _, a1, h1, d1 = p.grid(1)
        x0 = draws[0]
        u0 = np.asarray(Us[0])[nearest_idx(None, a0, h0, d0, x0)]
        w = draws[1]
        u1 = np.asarray(Us[1])[nearest_idx(None, a1, h1, d1, u0 + w)]
        err = u1 - x0
        return p.pw * u0 * u0 + err * err
    # problems/inventory.py:152-166 (stock snapped to the state grid each stage)
    g0 = p.state(0)
    x = g0[0][nearest_idx(None, g0[1], g0[2], g0[3], draws[0])]
    total = np.zeros(x.size)
    for mm in range(p.M):
        gm = p.grid(mm)
        u = np.asarray(Us[mm])[nearest_idx(None, gm[1], gm[2], gm[3], x)]
        w = draws[1 + mm]
        gn = p.state(mm + 1)
        x = gn[0][nearest_idx(None, gn[1], gn[2], gn[3], x + u - w)]
        total += p.oc * u + p.gamma(x)
    return total


# Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
# 1, 2, 3"), the device generator of device_monte_carlo_objective: restated
# here so its stream is checked bit for bit.  No reference analogue -- the
# reference draws with NumPy's PCG64, which the bitwise estimator uses.
_PH_M0, _PH_M1, _PH_W0, _PH_W1, _U32 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85, 0xFFFFFFFF


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    c = [np.asarray(v, dtype=np.uint64) & _U32 for v in (c0, c1, c2, c3)]
    k0, k1 = np.uint64(k0 & _U32), np.uint64(k1 & _U32)
    for _ in range(10):
        p0 = np.uint64(_PH_M0) * c[0]
        p1 = np.uint64(_PH_M1) * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ k0, p1 & np.uint64(_U32), (p0 >> np.uint64(32)) ^ c[3] ^ k1,
             p0 & np.uint64(_U32)]
        k0 = np.uint64((int(k0) + _PH_W0) & _U32)
        k1 = np.uint64((int(k1) + _PH_W1) & _U32)
    return [v.astype(np.uint32) for v in c]


def _u01(hi, lo):  # 53 bits -> (x + 0.5) * 2^-53, in (0, 1)
    x = ((hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)) >> np.uint64(11)
    return (x.astype(np.float64) + 0.5) * 2.0 ** -53


def philox_uniform01(seed, idx, c):
    """Unit uniforms U[i][2c], U[i][2c+1] of counter (idx, c), key = seed."""
    idx = np.asarray(idx, dtype=np.uint64)
    w = philox4x32_10(idx & np.uint64(_U32), idx >> np.uint64(32), np.full(idx.shape, c, np.uint64), 0,
                      seed & _U32, (seed >> 32) & _U32)
    return _u01(w[0], w[1]), _u01(w[2], w[3])


def philox_draws(p, seed, begin, end):
    """Device draw streams for samples [begin, end), in the reference's stream
    layout (csrc/ucp_mc.cuh: k_mc_draws).  Uniforms lo + (hi - lo) U[i][k]
    are bitwise; normals come from Box-Muller on (U[i][0], U[i][1]):
    r = sqrt(-2 ln u1), z = r cos(2 pi u2) and r sin(2 pi u2) -- the device's
    log/sincospi round differently from NumPy's, so normals agree to a few
    ulp, not bitwise."""
    idx = np.arange(begin, end, dtype=np.uint64)
    seed = int(seed) & ((1 << 64) - 1)

    def U(k):
        return philox_uniform01(seed, idx, k >> 1)[k & 1]

    def box_muller():
        u1, u2 = philox_uniform01(seed, idx, 0)
        r = np.sqrt(-2.0 * np.log(u1))
        return r * np.cos(2.0 * np.pi * u2), r * np.sin(2.0 * np.pi * u2)

    if p.name == "witsenhausen":
        zc, zs = box_muller()
        return np.stack([0.0 + p.sigma * zc, 0.0 + 1.0 * zs])
    if p.name == "zero_delay":
        return np.stack([0.0 + 1.0 * box_muller()[0], -1.0 + 2.0 * U(2)])
    return np.stack([-1.0 + 2.0 * U(s) for s in range(p.M + 1)])


def _shuffle_tree(a):
    """Lane 0 of a 32-lane __shfl_down tree (offsets 16..1) over the last axis."""
    a = a.copy()
    for off in (16, 8, 4, 2, 1):
        a[..., :off] = a[..., :off] + a[..., off:2 * off]
    return a[..., 0]


def mc_chunk_partials(values, chunk=4096, threads=256):
    """The device's fixed-order partial sum per chunk of ``values``: thread t
    sums elements t, t+threads, ... serially, lanes fold by shuffle tree,
    warps in order (csrc/ucp_mc.cuh: k_mc_partials)."""
    values = np.asarray(values, dtype=np.float64)
    nch = -(-values.size // chunk)
    v = np.zeros(nch * chunk)
    v[: values.size] = values
    v = v.reshape(nch, chunk // threads, threads)
    acc = np.zeros((nch, threads))
    for j in range(chunk // threads):
        acc = acc + v[:, j, :]
    warps = _shuffle_tree(acc.reshape(nch, threads // 32, 32))
    s = warps[:, 0]
    for w in range(1, threads // 32):
        s = s + warps[:, w]
    return s


def mc_reduce(partials, threads=1024):
    """k_mc_reduce's fixed-order sum of the chunk partials."""
    partials = np.asarray(partials, dtype=np.float64)
    rows = -(-partials.size // threads)
    v = np.zeros(max(rows, 1) * threads)
    v[: partials.size] = partials
    v = v.reshape(-1, threads)
    acc = np.zeros(threads)
    for r in range(v.shape[0]):
        acc = acc + v[r]
    warps = _shuffle_tree(acc.reshape(threads // 32, 32))
    s = warps[0]
    for w in range(1, threads // 32):
        s = s + warps[w]
    return float(s)


def mc_estimate(costs):
    """Estimate and stderr of the device estimator from per-sample costs,
    with the device's reduction order and two-pass variance."""
    costs = np.asarray(costs, dtype=np.float64)
    n = costs.size
    total = mc_reduce(mc_chunk_partials(costs))
    mean = total / n
    dev = costs - mean
    sq = mc_reduce(mc_chunk_partials(dev * dev))
    return total / n, math.sqrt(sq / (n - 1)) / math.sqrt(n)


def host_cpu_description() -> dict:
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "model": model}
