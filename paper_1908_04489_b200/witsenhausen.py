"""Witsenhausen's counterexample on the B200 (reference problems/witsenhausen.py).

    x1 = x0 + u0(y0),  y1 = x1 + w,  x2 = x1 - u1(y1),  cost = k^2 u0^2 + x2^2
    x0 ~ N(0, sigma^2),  w ~ N(0, 1),  y0 = x0

Stage-0 marginal cost (witsenhausen.py:62-70):
    C0(u, y) = f0(y) * (k^2 u^2 + sum_j W_j phi(y1_j - s) (s - u1_j)^2 + tails),  s = y + u
Stage-1 marginal cost (witsenhausen.py:71-78), the u1 estimator moments:
    C1(u, y) = A u^2 - 2 B u + C,  (A, B, C) = sum_i fw0_i phi(y - x1_i) (1, x1_i, x1_i^2)

All per-candidate work runs in libucp_b200 (csrc/ucp_kernels.cu) on
device-resident controllers; only the NumPy density constants (f0, fw0) and
the window bounds are computed on the host, once per problem.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from ._device import F64, I64, ptr, to_device_f64, to_device_i64
from .distributed import LOCAL, Sharding
from .grids import ControllerSet
from .numerics import Gaussian, pdf
from .device_problem import NO_ERROR, DeviceContext
from .problem import NumericError, Problem

__all__ = ["Witsenhausen"]

# below this many points shards are equal-sized (balancing would cost more than it saves)
BALANCE_MIN_POINTS = int(os.environ.get("UCP_BALANCE_MIN_POINTS", 1 << 14))
# replay block iterations from CUDA graphs (UCP_GRAPHS=0 disables)
GRAPH_BLOCKS = os.environ.get("UCP_GRAPHS", "1") != "0"

class _WcDevice(DeviceContext):
    """Device-resident constants and ABI struct of one Witsenhausen problem
    (plus the shared workspace / error log / window cache)."""

    def graph_state(self) -> dict:
        """Fixed-address buffers of the graph-replayed block executor."""
        if self._graph_state is None:
            d0, d1 = int(self.y0.numel()), int(self.y1.numel())
            self._graph_state = {
                "u0": torch.empty(d0, dtype=F64, device=self.device),
                "u1": torch.empty(d1, dtype=F64, device=self.device),
                "s0": torch.empty(d0, dtype=F64, device=self.device),
                "s1": torch.empty(d1, dtype=F64, device=self.device),
                "err": torch.full((6,), NO_ERROR, dtype=I64, device=self.device),
            }
        return self._graph_state

    def block_params(self, cfg, g0, g1):
        """ucp_local_params[2] for both stages, cached per config (stable address and bits)."""
        key = (cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g0), cfg.cap_for(g1))
        if key not in self._lp_cache:
            self._lp_cache[key] = (_lib.LocalParams * 2)(
                *[_lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g)) for g in (g0, g1)])
        return self._lp_cache[key]

    def __init__(self, prob: "Witsenhausen", device=None):
        super().__init__(prob, device)
        self._graph_state = None
        self._lp_cache: dict = {}
        g0, g1 = prob.grids
        self.y0 = to_device_f64(g0.points, self.device)
        self.y1 = to_device_f64(g1.points, self.device)
        self.f0 = to_device_f64(prob._f0, self.device)
        self.fw0 = to_device_f64(prob._fw0, self.device)
        self.P = _lib.WcProblem(prob.k, g0.a, g0.spacing, g0.d, g1.a, g1.spacing, g1.d,
                                ptr(self.y0), ptr(self.y1), ptr(self.f0), ptr(self.fw0),
                                {"reference": 0, "fma": _lib.WC_FAST,
                                 "table": _lib.WC_FAST | _lib.WC_TABLE}[prob.arithmetic])


class Witsenhausen(Problem):
    name = "witsenhausen"

    ARITHMETIC = ("reference", "fma", "table")

    def __init__(self, k: float = 0.2, sigma: float = 5.0, grids=None, device=None, arithmetic: str = "reference"):
        """``arithmetic``: "reference" (default) evaluates every stage-0 walk in
        the reference's exact operation order -- results bitwise the reference's;
        "fma" is the opt-in, tolerance-stated fast mode (h folded into the pdf
        recurrence, FMA in the v-weighted sums: 6 instead of 8 FP64 instructions
        per walk node; costs equal to rounding, argmin picks may differ on
        near-ties -- tests/test_gpu_fast_mode.py states the tolerance);
        "table" (grids with h1 <= 2e-3) evaluates window sums from
        expansions, O(1) per candidate: per-cell Taylor expansions in both
        stage-0 phases and the objective (the reference walk's rounding bias
        reproduced), per-tile Taylor expansions of the stage-1 moments
        (DESIGN.md §2b states the tolerance: J of a snapshot within 1e-9,
        near-tie picks, converged J within 1e-9)."""
        if arithmetic not in self.ARITHMETIC:
            raise ValueError(f"witsenhausen.arithmetic must be one of {self.ARITHMETIC} (got {arithmetic!r})")
        self.arithmetic = arithmetic
        if not k > 0.0:
            raise ValueError(f"witsenhausen.k must be positive (got {k})")
        if not sigma > 0.0:
            raise ValueError(f"witsenhausen.sigma must be positive (got {sigma})")
        self.k = float(k)
        self.sigma = float(sigma)
        super().__init__(grids)
        self._state_density = Gaussian(0.0, self.sigma)
        g0 = self.grids[0]
        # host NumPy constants, exactly as the reference (witsenhausen.py:47-53)
        self._f0 = pdf(self._state_density, g0.points)
        w0 = np.full(g0.d, g0.spacing)
        w0[0] *= 0.5
        w0[-1] *= 0.5
        self._fw0 = w0 * self._f0
        self._device_arg = device
        self._dev: _WcDevice | None = None

    def default_grid_specs(self):
        return [(-25.0, 25.0, 2000), (-25.0, 25.0, 2000)]

    # ------------------------------------------------------------- device
    def device_context(self) -> _WcDevice:
        if self._dev is None:
            self._dev = _WcDevice(self, self._device_arg)
        return self._dev

    @property
    def device(self) -> torch.device:
        return self.device_context().device

    def _override_host_constants(self, f0, fw0) -> None:
        """Replace the host-NumPy densities (parity tests replaying a reference
        run made on another host's NumPy); must precede first device use."""
        if self._dev is not None:
            raise RuntimeError("device context already created")
        self._f0 = np.ascontiguousarray(f0, dtype=np.float64)
        self._fw0 = np.ascontiguousarray(fw0, dtype=np.float64)

    def _uv(self, U: ControllerSet):
        dev = self.device_context().device
        return U.device_values(0, dev), U.device_values(1, dev)

    # ------------------------------------------------- plugin API (host I/O)
    def marginal_cost_segmented(self, m, u_flat, offsets, y_centers, U):
        """witsenhausen.py:59-79; host arrays in, host array out."""
        if m not in (0, 1):
            raise ValueError(f"stage index {m} out of range for {self.name}")
        D = self.device_context()
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        y_centers = np.ascontiguousarray(y_centers, dtype=np.float64)
        u_flat = np.ascontiguousarray(u_flat, dtype=np.float64)
        nseg = offsets.size - 1
        if nseg != y_centers.size:
            raise ValueError("offsets and y_centers disagree")
        n = int(offsets[-1]) if nseg >= 0 else 0
        out = torch.empty(max(n, 1), dtype=F64, device=D.device)
        if n:
            u0, u1 = self._uv(U)
            ud = to_device_f64(u_flat, D.device)
            od = to_device_i64(offsets, D.device)
            yd = to_device_f64(y_centers, D.device)
            if m == 0:
                f0 = to_device_f64(pdf(self._state_density, y_centers), D.device)
                _lib.call("ucp_wc_stage0_cost_ws", ctypes.byref(D.P), ptr(u1), ptr(ud), n, ptr(od), ptr(yd),
                          ptr(f0), nseg, ptr(out), D.ws, D.stream)
            else:
                _lib.call("ucp_wc_stage1_cost", ctypes.byref(D.P), ptr(u0), ptr(ud), n, ptr(od), ptr(yd),
                          nseg, ptr(out), D.ws, D.stream)
        return out[:n].cpu().numpy()

    # ------------------------------------------------ solver sweeps (device)
    # ---- work-balanced shards (multi-GPU) --------------------------------
    # Plans are cached per (stage, weighting) and refreshed at the objective's
    # synchronisation (device_objective): the cuts are computed on the device
    # from that snapshot and read back in the same copy as J, so a phase never
    # waits on the host for its plan.  A phase uses the plan of the latest
    # objective snapshot (the first use per problem computes it directly).
    # Boundaries never change a result bit, only the balance.
    # Balanced-plan walks stop at their no-op tail about 8.5 sigma past the
    # centre (the throughput walk's tail exit: 83% of the full windows' nodes at
    # the bench snapshot), so a walk's cost is its clamped [s - 12, s + 8.5]
    # span, not the full window; shard_projection measured 17% exhaustion
    # imbalance at 8 ranks with full windows.
    WALK_TAIL_SIGMAS = 8.5 if os.environ.get("UCP_TAIL_EXIT", "1") != "0" else 12.0

    def _plan_weights(self, key, U: ControllerSet) -> torch.Tensor:
        """Per-point work estimates of plan ``key`` = (stage, scaled): walk nodes
        for stage 0 (times the number of distinct-by-run window candidates for
        exhaustion, the ones the kernels evaluate), in-range support points for
        stage 1.  Every rank derives them from the same snapshot."""
        m, scaled = key
        D = self.device_context()
        u0, _ = self._uv(U)
        g1 = self.grids[1]
        if m == 0:
            s = D.y0 + u0
            span = torch.clamp(torch.minimum(s + self.WALK_TAIL_SIGMAS, torch.full_like(s, g1.b))
                               - torch.maximum(s - 12.0, torch.full_like(s, g1.a)), min=0.0)
            w = (span / g1.spacing).to(torch.int64) + 1
            if scaled is not None:
                lo, hi = D.window(self, 0, scaled)
                runs = torch.zeros_like(lo)
                runs[1:] = torch.cumsum((u0[1:] != u0[:-1]).to(torch.int64), 0)
                w = w * (1 + runs[hi] - runs[lo])
            return w
        return self._moments_weights(D.y0 + u0, D.y1)

    @staticmethod
    def _moments_weights(x1: torch.Tensor, yq: torch.Tensor, tile: int = 256, qblock: int = 128) -> torch.Tensor:
        """Stage-1 work per query as the moments kernels do it: a 128-query block
        (ascending grid queries) visits every 256-point support tile (index
        order) whose [min, max] of x1 comes within 12 of the block's span, all
        256 pairs of a visited tile (k_moments' tile skipping).  live =
        #{tiles: max >= ymin - 12} - #{tiles: min > ymax + 12} (min <= max), two
        sorted counts instead of a block x tile matrix; a NaN in a tile keeps it
        live.  Returns int64 pairs per query."""
        d0, d1 = x1.numel(), yq.numel()
        nt = -(-d0 // tile)
        pad = nt * tile - d0
        nan = torch.isnan(x1)
        lo = torch.nn.functional.pad(torch.where(nan, torch.full_like(x1, -torch.inf), x1), (0, pad),
                                     value=torch.inf).view(nt, tile).amin(1)
        hi = torch.nn.functional.pad(torch.where(nan, torch.full_like(x1, torch.inf), x1), (0, pad),
                                     value=-torch.inf).view(nt, tile).amax(1)
        nb = -(-d1 // qblock)
        first = torch.arange(nb, device=yq.device) * qblock
        ymin, ymax = yq[first], yq[torch.clamp(first + qblock - 1, max=d1 - 1)]
        reach_lo = nt - torch.searchsorted(torch.sort(hi).values, ymin - 12.0)           # tiles with max >= ymin-12
        past_hi = nt - torch.searchsorted(torch.sort(lo).values, ymax + 12.0, right=True)  # tiles with min > ymax+12
        live = torch.clamp(reach_lo - past_hi, min=1)
        return torch.repeat_interleave(live * tile, qblock)[:d1]

    def _plan(self, m: int, U: ControllerSet, sharding: Sharding, radius=None) -> tuple:
        """Shard boundaries for a stage-m phase (``radius``: stage-0 exhaustion
        windows of that radius weight the walks)."""
        d = self.grids[m].d
        if sharding.world == 1 or d < BALANCE_MIN_POINTS:
            return sharding.equal_plan(d) if sharding.world > 1 else (0, d)
        key = (m, radius if m == 0 else None)
        cache = self.device_context().plans
        if (key, sharding.world) not in cache:  # first use: computed now (one read-back)
            cache[(key, sharding.world)] = sharding.plan(d, self._plan_weights(key, U))
        return cache[(key, sharding.world)]

    def _queue_plan_refresh(self, U: ControllerSet, sharding: Sharding):
        """Device cuts of every cached plan for snapshot U (no synchronisation);
        returns (keys, int64 tensor) for _apply_plan_refresh."""
        keys = [k for k in self.device_context().plans if k[1] == sharding.world]
        if not keys or sharding.world == 1:
            return [], None
        cuts = torch.cat([sharding.plan_cuts(self._plan_weights(k, U)) for k, _ in keys])
        return keys, cuts

    def _apply_plan_refresh(self, keys, host_cuts, sharding: Sharding) -> None:
        n = sharding.world - 1
        cache = self.device_context().plans
        for q, key in enumerate(keys):
            cache[key] = sharding.plan_from_cuts(self.grids[key[0][0]].d, host_cuts[q * n:(q + 1) * n])

    def device_local_update(self, m: int, U: ControllerSet, cfg, sharding: Sharding = LOCAL):
        """One local-update sweep of stage m (solver.py:179-203); returns a CUDA tensor."""
        D = self.device_context()
        g = self.grids[m]
        u0, u1 = self._uv(U)
        lp = _lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g))
        bounds = self._plan(m, U, sharding)
        begin, end = sharding.shard(bounds)
        buf = sharding.padded_buffer(bounds, D.device)
        err = D.errors.slot("local", m, sharding)
        _lib.call("ucp_wc_local_update", ctypes.byref(D.P), m, ptr(u0), ptr(u1), ctypes.byref(lp), begin, end,
                  sharding.rank_ptr(buf, bounds), ptr(err), D.ws, D.stream)
        return sharding.gather(buf, bounds, g.d)

    def device_exhaustion(self, m: int, U: ControllerSet, cfg, sharding: Sharding = LOCAL):
        """One partial-exhaustion sweep of stage m (solver.py:206-223)."""
        D = self.device_context()
        g = self.grids[m]
        u0, u1 = self._uv(U)
        lo, hi = D.window(self, m, cfg.radius_for(g))
        bounds = self._plan(m, U, sharding, radius=cfg.radius_for(g) if m == 0 else None)
        begin, end = sharding.shard(bounds)
        buf = sharding.padded_buffer(bounds, D.device)
        err = D.errors.slot("exhaustion", m, sharding)
        bound = D.candidate_bound(self, m, cfg.radius_for(g), begin, end) if m == 0 else 0
        _lib.call("ucp_wc_exhaustion", ctypes.byref(D.P), m, ptr(u0), ptr(u1), ptr(lo), ptr(hi), bound, begin, end,
                  sharding.rank_ptr(buf, bounds), ptr(err), D.ws, D.stream)
        return sharding.gather(buf, bounds, g.d)

    def device_run_block(self, kind: str, iters: int, U: ControllerSet, cfg, graphs: bool = True) -> ControllerSet:
        """`iters` iterations of one phase kind over both stages in ONE native
        call (solver.py:226-231), unsharded.  With ``graphs`` the iterations
        after the first replay a CUDA graph captured once per block signature
        (fixed per-problem state buffers), which removes the per-kernel launch
        cost that dominates small grids."""
        from .grids import SampledController

        if iters <= 0:
            return U
        D = self.device_context()
        u0, u1 = self._uv(U)
        g0, g1 = self.grids
        lp = D.block_params(cfg, g0, g1)
        if kind == "local":
            code, wins, bound = 0, (None, None, None, None), 0
        else:
            code = 1
            lo0, hi0 = D.window(self, 0, cfg.radius_for(g0))
            lo1, hi1 = D.window(self, 1, cfg.radius_for(g1))
            wins = (ptr(lo0), ptr(hi0), ptr(lo1), ptr(hi1))
            bound = D.candidate_bound(self, 0, cfg.radius_for(g0), 0, g0.d)
        if graphs and iters > 1 and GRAPH_BLOCKS:
            st = D.graph_state()
            st["u0"].copy_(u0)
            st["u1"].copy_(u1)
            _lib.call("ucp_wc_run_block_graph", ctypes.byref(D.P), code, int(iters), ptr(st["u0"]), ptr(st["u1"]), lp,
                      *wins, bound, ptr(st["s0"]), ptr(st["s1"]), ptr(st["err"]), D.ws, D.stream)
            rows = D.errors.slots([("block", 0, (kind, iters, U, cfg)), ("block", 1, (kind, iters, U, cfg))], LOCAL)
            rows.view(-1).copy_(st["err"])
            st["err"].fill_(NO_ERROR)
            out0, out1 = st["u0"].clone(), st["u1"].clone()
        else:
            out0, out1 = u0.clone(), u1.clone()
            s0, s1 = torch.empty_like(out0), torch.empty_like(out1)
            err = D.errors.slots([(kind, m) for _ in range(iters) for m in (0, 1)], LOCAL)
            _lib.call("ucp_wc_run_block", ctypes.byref(D.P), code, int(iters), ptr(out0), ptr(out1), lp, *wins,
                      bound, ptr(s0), ptr(s1), ptr(err), D.ws, D.stream)
        return ControllerSet((SampledController(g0, out0, _trusted_device=True),
                              SampledController(g1, out1, _trusted_device=True)))

    def _replay_block_error(self, payload, sharding) -> None:
        """Re-run a graph-replayed block eagerly (per-phase error slots) and raise its first failure."""
        kind, iters, U, cfg = payload
        self.device_run_block(kind, iters, U, cfg, graphs=False)
        self.device_context().errors.flush(sharding)

    def _queue_objective(self, U: ControllerSet, sharding: Sharding, err: torch.Tensor) -> torch.Tensor:
        """Queue the objective of U (problem.py:110-127: stage-0 integrand, then
        the serial trapezoid); returns a device int64[1] holding J's bits, the
        first non-finite integrand point goes to ``err`` (atomicMin)."""
        self.check_controllers(U)
        D = self.device_context()
        g = self.grids[0]
        u0, u1 = self._uv(U)
        bounds = self._plan(0, U, sharding)
        begin, end = sharding.shard(bounds)
        buf = sharding.padded_buffer(bounds, D.device)
        jbits = torch.empty(1, dtype=I64, device=D.device)
        _lib.call("ucp_wc_objective_terms_ws", ctypes.byref(D.P), ptr(u0), ptr(u1), begin, end,
                  sharding.rank_ptr(buf, bounds), err.data_ptr(), D.ws, D.stream)
        terms = sharding.gather(buf, bounds, g.d)
        sharding.allreduce_min_(err)
        _lib.call("ucp_trapezoid_sum", ptr(terms), g.d, g.spacing, jbits.data_ptr(), None, D.stream)
        return jbits

    def device_objective_terms(self, U: ControllerSet, sharding: Sharding = LOCAL) -> torch.Tensor:
        """The objective's per-point integrand c_i = C0(u0_i, y_i) (problem.py:119-126)
        as a device tensor of d0 doubles -- the values the serial trapezoid sums.
        Non-finite terms are reported like device_objective's."""
        D = self.device_context()
        res = torch.full((1,), NO_ERROR, dtype=I64, device=D.device)
        self.check_controllers(U)
        g = self.grids[0]
        u0, u1 = self._uv(U)
        bounds = self._plan(0, U, sharding)
        begin, end = sharding.shard(bounds)
        buf = sharding.padded_buffer(bounds, D.device)
        _lib.call("ucp_wc_objective_terms_ws", ctypes.byref(D.P), ptr(u0), ptr(u1), begin, end,
                  sharding.rank_ptr(buf, bounds), res.data_ptr(), D.ws, D.stream)
        terms = sharding.gather(buf, bounds, g.d)
        sharding.allreduce_min_(res)
        bad = int(D.errors.flush(sharding, extra=res)[0])
        if bad != NO_ERROR:
            raise NumericError(
                f"{self.name}: non-finite objective integrand at stage 0, grid point {bad} "
                f"(y={g.points[bad]!r}, u={U.values(0)[bad]!r})")
        return terms

    def device_objective(self, U: ControllerSet, sharding: Sharding = LOCAL, deferred=()) -> float:
        """problem.py:110-127 on the device.  ``deferred`` objectives (from
        device_objective_deferred) are read in the same synchronisation."""
        D = self.device_context()
        res = torch.full((1,), NO_ERROR, dtype=I64, device=D.device)
        jbits = self._queue_objective(U, sharding, res)
        keys, cuts = self._queue_plan_refresh(U, sharding)
        # one synchronisation: the pending phase-error rows (deferred objectives
        # among them, in queue order), every J and the refreshed shard plans
        # travel together
        extra = torch.cat([res, jbits] + [p[0] for p in deferred] + ([cuts] if keys else []))
        host = D.errors.flush(sharding, extra=extra)
        if keys:
            nj = 2 + len(deferred)
            self._apply_plan_refresh(keys, host[nj:], sharding)
            host = host[:nj]
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
        """Queue the objective of U without synchronising; its failure is
        raised in queue order by the next synchronisation, and its value is
        read by the next device_objective(..., deferred=[handle])."""
        D = self.device_context()
        row = D.errors.slots([("objective", 0, U)], sharding)[0]
        jbits = self._queue_objective(U, sharding, row[:1])
        return (jbits, [])

    def flush_errors(self, sharding: Sharding = LOCAL) -> None:
        if self._dev is not None:
            self._dev.errors.flush(sharding)

    def objective(self, U) -> float:
        return self.device_objective(U)
