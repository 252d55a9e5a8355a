"""Config 5 -- the paper's additional UCP examples on the B200.

* ``ZeroDelay`` (reference problems/zero_delay.py): zero-delay source-channel
  coding with uniform channel noise; 2 stages.
* ``Inventory`` (reference problems/inventory.py): multi-stage (M >= 1)
  inventory control with nonnegative orders.

Both run their sweeps with the generic device kernels of
csrc/ucp_config5.cuh (cost functors over the exact cell-overlap integrals);
the solver loop, API and error behaviour are the Witsenhausen path's.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._device import F64, I64, ptr, to_device_f64, to_device_i64
from .device_problem import NO_ERROR, DeviceContext
from .distributed import LOCAL, Sharding
from .grids import ControllerSet, content_key
from .numerics import Gaussian, pdf
from .problem import NumericError, Problem

__all__ = ["ZeroDelay", "Inventory"]

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
MAX_STAGES = 16


class ZdProblemC(ctypes.Structure):
    """struct ucp_zd_problem"""

    _fields_ = [("power_weight", c_dbl), ("a0", c_dbl), ("h0", c_dbl), ("d0", c_i64), ("a1", c_dbl),
                ("h1", c_dbl), ("d1", c_i64), ("y0", c_vp), ("y1", c_vp), ("f0", c_vp), ("fw0", c_vp)]


class InvProblemC(ctypes.Structure):
    """struct ucp_inv_problem"""

    _fields_ = [("stages", c_i32), ("quadratic", c_i32), ("order_cost", c_dbl), ("holding_rate", c_dbl),
                ("backlog_rate", c_dbl), ("a", c_dbl * MAX_STAGES), ("h", c_dbl * MAX_STAGES),
                ("d", c_i64 * MAX_STAGES), ("pts", c_vp * MAX_STAGES), ("ukey", c_vp)]


_PP = ctypes.POINTER
_SIGS = {
    "ucp_unif_moments_grid": (ctypes.c_int, [c_vp, c_i64, c_vp, c_dbl, c_dbl, c_i64, c_dbl, c_vp, c_vp, c_vp, c_vp]),
    "ucp_unif_ball_sum": (ctypes.c_int, [c_vp, c_i64, c_vp, c_dbl, c_dbl, c_i64, c_dbl, c_vp, c_vp]),
    "ucp_unif_propagate": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_i64, c_dbl, c_vp, c_vp]),
    "ucp_unif_moments_points": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_i64, c_dbl,
                                               c_vp, c_vp, c_vp, c_vp]),
    "ucp_zd_cost": (ctypes.c_int, [_PP(ZdProblemC), ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                   c_vp, c_vp, c_vp]),
    "ucp_zd_local_update": (ctypes.c_int, [_PP(ZdProblemC), ctypes.c_int, c_vp, c_vp, _PP(_lib.LocalParams), c_i64,
                                           c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ucp_zd_exhaustion": (ctypes.c_int, [_PP(ZdProblemC), ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                                         c_vp, c_vp, c_vp, c_vp]),
    "ucp_zd_objective_terms": (ctypes.c_int, [_PP(ZdProblemC), c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "ucp_inv_cost": (ctypes.c_int, [_PP(InvProblemC), ctypes.c_int, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp,
                                    c_vp, c_vp]),
    "ucp_inv_local_update": (ctypes.c_int, [_PP(InvProblemC), ctypes.c_int, c_vp, _PP(_lib.LocalParams), c_i64,
                                            c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ucp_inv_exhaustion": (ctypes.c_int, [_PP(InvProblemC), ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                                          c_vp, c_vp, c_vp, c_vp]),
    "ucp_inv_objective_terms": (ctypes.c_int, [_PP(InvProblemC), c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ucp_inv_forward_density": (ctypes.c_int, [_PP(InvProblemC), ctypes.c_int, c_vp, c_vp, c_vp, c_vp]),
}
_lib.SIGNATURES.update(_SIGS)


def _bind():
    lib = _lib.load()
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


class _DeviceSweeps:
    """Device sweeps shared by the config-5 problems (same contract as
    Witsenhausen.device_*: sharded over [begin, end), one all-gather)."""

    _dev: DeviceContext | None

    def device_context(self) -> DeviceContext:
        if self._dev is None:
            _bind()
            self._dev = DeviceContext(self, self._device_arg)
            self._build_structs()
        return self._dev

    @property
    def device(self):
        return self.device_context().device

    def _uptrs(self, U: ControllerSet):
        dev = self.device_context().device
        ts = [U.device_values(m, dev) for m in range(self.M)]
        return ts

    def flush_errors(self, sharding: Sharding = LOCAL) -> None:
        if self._dev is not None:
            self._dev.errors.flush(sharding)

    def _sweep(self, kind, m, U, cfg, sharding):
        D = self.device_context()
        g = self.grids[m]
        ts = self._uptrs(U)
        begin, end = sharding.bounds(g.d)
        buf = sharding.out_buffer(g.d, D.device)
        err = D.errors.slot(kind, m, sharding)
        if kind == "local":
            lp = _lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g))
            self._abi_local(m, ts, lp, begin, end, buf, err)
        else:
            lo, hi = D.window(self, m, cfg.radius_for(g))
            self._abi_exhaustion(m, ts, lo, hi, D.window_width(self, m, cfg.radius_for(g)), begin, end, buf, err)
        sharding.allgather_(buf)
        return buf[: g.d]

    def device_local_update(self, m, U, cfg, sharding: Sharding = LOCAL):
        return self._sweep("local", m, U, cfg, sharding)

    def device_exhaustion(self, m, U, cfg, sharding: Sharding = LOCAL):
        return self._sweep("exhaustion", m, U, cfg, sharding)

    def _queue_objective(self, U: ControllerSet, sharding: Sharding, err: torch.Tensor) -> torch.Tensor:
        """Queue the objective (problem.py:110-127: stage-0 integrand + serial
        trapezoid); returns device int64[1] with J's bits, first bad point -> err."""
        self.check_controllers(U)
        D = self.device_context()
        g = self.grids[0]
        ts = self._uptrs(U)
        begin, end = sharding.bounds(g.d)
        terms = sharding.out_buffer(g.d, D.device)
        jbits = torch.empty(1, dtype=I64, device=D.device)
        self._abi_terms(ts, begin, end, terms, err)
        sharding.allgather_(terms)
        sharding.allreduce_min_(err)
        _lib.call("ucp_trapezoid_sum", ptr(terms), g.d, g.spacing, jbits.data_ptr(), None, D.stream)
        return jbits

    def device_objective(self, U: ControllerSet, sharding: Sharding = LOCAL, deferred=()) -> float:
        """problem.py:110-127 on the device; ``deferred`` objectives (from
        device_objective_deferred) are read in the same synchronisation."""
        D = self.device_context()
        res = torch.full((1,), NO_ERROR, dtype=I64, device=D.device)
        jbits = self._queue_objective(U, sharding, res)
        host = D.errors.flush(sharding, extra=torch.cat([res, jbits] + [p[0] for p in deferred]))
        bad = int(host[0])
        if bad != NO_ERROR:
            g = self.grids[0]
            raise NumericError(
                f"{self.name}: non-finite objective integrand at stage 0, grid point {bad} "
                f"(y={g.points[bad]!r}, u={U.values(0)[bad]!r})")
        vals = host[1:].view(np.float64)
        for p, v in zip(deferred, vals[1:]):
            p[1].append(float(v))
        return float(vals[0])

    def device_objective_deferred(self, U: ControllerSet, sharding: Sharding = LOCAL):
        """Queue the objective without synchronising (see Witsenhausen)."""
        D = self.device_context()
        row = D.errors.slots([("objective", 0, U)], sharding)[0]
        return (self._queue_objective(U, sharding, row[:1]), [])

    def objective(self, U) -> float:
        return self.device_objective(U)

    def marginal_cost_segmented(self, m, u_flat, offsets, y_centers, U):
        if not 0 <= m < self.M:
            raise ValueError(f"stage index {m} out of range for {self.name}")
        D = self.device_context()
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        y_centers = np.ascontiguousarray(y_centers, dtype=np.float64)
        u_flat = np.ascontiguousarray(u_flat, dtype=np.float64)
        nseg = offsets.size - 1
        n = int(offsets[-1]) if nseg >= 0 else 0
        out = torch.empty(max(n, 1), dtype=F64, device=D.device)
        if n:
            ts = self._uptrs(U)
            self._abi_cost(m, ts, to_device_f64(u_flat, D.device), n, to_device_i64(offsets, D.device),
                           to_device_f64(y_centers, D.device), y_centers, nseg, out)
        return out[:n].cpu().numpy()


class ZeroDelay(_DeviceSweeps, Problem):
    """zero_delay.py:36-86; f0 and fw0 are host NumPy constants (uploaded)."""

    name = "zero_delay"

    def __init__(self, power_weight: float = 2.0, grids=None, device=None):
        if not power_weight > 0.0:
            raise ValueError(f"zero_delay.power_weight must be positive (got {power_weight})")
        self.power_weight = float(power_weight)
        super().__init__(grids)
        self._source = Gaussian(0.0, 1.0)
        g0 = self.grids[0]
        self._f0 = pdf(self._source, g0.points)
        w0 = np.full(g0.d, g0.spacing)
        w0[0] *= 0.5
        w0[-1] *= 0.5
        self._fw0 = w0 * self._f0
        self._device_arg = device
        self._dev = None

    def default_grid_specs(self):
        return [(-5.0, 5.0, 2000), (-6.0, 6.0, 2000)]

    def derivatives_batch(self, m, u, y, U, h):
        # zero_delay.py:56-65: probe at least one decoder cell wide (the device
        # local update applies the same floor)
        return super().derivatives_batch(m, u, y, U, np.maximum(h, self.grids[1].spacing))

    def _override_host_constants(self, f0, fw0):
        if self._dev is not None:
            raise RuntimeError("device context already created")
        self._f0 = np.ascontiguousarray(f0, dtype=np.float64)
        self._fw0 = np.ascontiguousarray(fw0, dtype=np.float64)

    def _build_structs(self):
        dev = self._dev.device
        g0, g1 = self.grids
        self._t = [to_device_f64(x, dev) for x in (g0.points, g1.points, self._f0, self._fw0)]
        self._P = ZdProblemC(self.power_weight, g0.a, g0.spacing, g0.d, g1.a, g1.spacing, g1.d,
                             *(ptr(t) for t in self._t))

    def _abi_local(self, m, ts, lp, begin, end, buf, err):
        D = self._dev
        _lib.call("ucp_zd_local_update", ctypes.byref(self._P), m, ptr(ts[0]), ptr(ts[1]), ctypes.byref(lp), begin,
                  end, ptr(buf), ptr(err), D.ws, D.stream)

    def _abi_exhaustion(self, m, ts, lo, hi, wmax, begin, end, buf, err):
        D = self._dev
        _lib.call("ucp_zd_exhaustion", ctypes.byref(self._P), m, ptr(ts[0]), ptr(ts[1]), ptr(lo), ptr(hi), wmax,
                  begin, end, ptr(buf), ptr(err), D.ws, D.stream)

    def _abi_terms(self, ts, begin, end, terms, err):
        _lib.call("ucp_zd_objective_terms", ctypes.byref(self._P), ptr(ts[0]), ptr(ts[1]), begin, end, ptr(terms),
                  err.data_ptr(), self._dev.stream)

    def _abi_cost(self, m, ts, ud, n, od, yd, y_host, nseg, out):
        D = self._dev
        f0 = to_device_f64(pdf(self._source, y_host), D.device) if m == 0 else yd
        _lib.call("ucp_zd_cost", ctypes.byref(self._P), m, ptr(ts[0]), ptr(ts[1]), ptr(ud), n, ptr(od), ptr(yd),
                  ptr(f0), nseg, ptr(out), D.ws, D.stream)


_STAGE_COSTS = ("piecewise_linear", "quadratic")


class Inventory(_DeviceSweeps, Problem):
    """inventory.py:31-150: M-stage inventory, uniform demand, orders >= 0."""

    name = "inventory"

    def __init__(self, stages: int = 2, order_cost: float = 0.1, stage_cost: str = "piecewise_linear",
                 holding_rate: float = 1.0, backlog_rate: float = 1.0, grids=None, device=None):
        if int(stages) != stages or stages < 1:
            raise ValueError(f"inventory.stages must be a positive integer (got {stages})")
        if stages > MAX_STAGES:
            raise ValueError(f"inventory.stages must be at most {MAX_STAGES} on the device (got {stages})")
        if order_cost < 0.0:
            raise ValueError(f"inventory.order_cost must be nonnegative (got {order_cost})")
        if stage_cost not in _STAGE_COSTS:
            raise ValueError(f"inventory.stage_cost must be one of {_STAGE_COSTS} (got {stage_cost!r})")
        if stage_cost == "piecewise_linear" and not (holding_rate > 0.0 and backlog_rate > 0.0):
            raise ValueError("inventory holding/backlog rates must be positive")
        self.stages = int(stages)
        self.order_cost = float(order_cost)
        self.stage_cost = stage_cost
        self.holding_rate = float(holding_rate)
        self.backlog_rate = float(backlog_rate)
        super().__init__(grids)
        self._device_arg = device
        self._dev = None
        self.reuse = True  # reuse densities / costs-to-go of unchanged stages (result-identical)

    def default_grid_specs(self):
        return [(-3.0, 3.0, 601)] * self.stages

    def _state_grid(self, mm):  # inventory.py:74-76
        return self.grids[min(mm, self.stages - 1)]

    def derivatives_batch(self, m, u, y, U, h):
        # inventory.py:131-136: probe at least one next-stage state cell wide
        return super().derivatives_batch(m, u, y, U, np.maximum(h, self._state_grid(m + 1).spacing))

    def gamma(self, x):
        x = np.asarray(x, dtype=np.float64)
        if self.stage_cost == "quadratic":
            out = x * x
        else:
            out = self.holding_rate * np.maximum(x, 0.0) + self.backlog_rate * np.maximum(-x, 0.0)
        return float(out) if out.ndim == 0 else out

    def project(self, m, values):
        return np.maximum(values, 0.0)

    def project_device(self, m, t: torch.Tensor) -> torch.Tensor:
        """np.maximum(t, 0.0) with NumPy's NaN/zero semantics, on device."""
        return torch.where((t > 0.0) | torch.isnan(t), t, torch.zeros_like(t))

    def _build_structs(self):
        dev = self._dev.device
        self._t = [to_device_f64(g.points, dev) for g in self.grids]
        P = InvProblemC()
        P.stages = self.stages
        P.quadratic = 1 if self.stage_cost == "quadratic" else 0
        P.order_cost, P.holding_rate, P.backlog_rate = self.order_cost, self.holding_rate, self.backlog_rate
        for m, g in enumerate(self.grids):
            P.a[m], P.h[m], P.d[m], P.pts[m] = g.a, g.spacing, g.d, ptr(self._t[m])
        self._P = P

    def _uarray(self, ts):
        """Device pointers of the controllers, and their content keys into
        the problem struct (the library then reuses densities / costs-to-go
        of unchanged stages across calls; no keys, no reuse)."""
        arr = (c_vp * MAX_STAGES)(*[ptr(t) for t in ts])
        keys = [content_key(t) for t in ts]
        if self.reuse and all(keys):
            self._ukeys = (ctypes.c_uint64 * MAX_STAGES)(*keys)
            self._P.ukey = ctypes.cast(self._ukeys, c_vp)
        else:
            self._P.ukey = None
        return arr

    def _abi_local(self, m, ts, lp, begin, end, buf, err):
        D = self._dev
        _lib.call("ucp_inv_local_update", ctypes.byref(self._P), m, ctypes.cast(self._uarray(ts), c_vp),
                  ctypes.byref(lp), begin, end, ptr(buf), ptr(err), D.ws, D.stream)

    def _abi_exhaustion(self, m, ts, lo, hi, wmax, begin, end, buf, err):
        D = self._dev
        _lib.call("ucp_inv_exhaustion", ctypes.byref(self._P), m, ctypes.cast(self._uarray(ts), c_vp), ptr(lo),
                  ptr(hi), wmax, begin, end, ptr(buf), ptr(err), D.ws, D.stream)

    def _abi_terms(self, ts, begin, end, terms, err):
        D = self._dev
        _lib.call("ucp_inv_objective_terms", ctypes.byref(self._P), ctypes.cast(self._uarray(ts), c_vp), begin, end,
                  ptr(terms), err.data_ptr(), D.ws, D.stream)

    def _abi_cost(self, m, ts, ud, n, od, yd, y_host, nseg, out):
        D = self._dev
        _lib.call("ucp_inv_cost", ctypes.byref(self._P), m, ctypes.cast(self._uarray(ts), c_vp), ptr(ud), n,
                  ptr(od), ptr(yd), nseg, ptr(out), D.ws, D.stream)

    def forward_density(self, m, U) -> np.ndarray:
        """Stock density at stage m (inventory.py:96-110), computed on device."""
        if not 0 <= m < self.stages:
            raise ValueError(f"stage index {m} out of range for {self.name}")
        D = self.device_context()
        ts = self._uptrs(U)
        out = torch.empty(self.grids[m].d, dtype=F64, device=D.device)
        _lib.call("ucp_inv_forward_density", ctypes.byref(self._P), m, ctypes.cast(self._uarray(ts), c_vp),
                  ptr(out), D.ws, D.stream)
        return out.cpu().numpy()
