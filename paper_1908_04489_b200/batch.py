"""Batched multi-instance engine (config 4).

``solve_batch`` solves B Witsenhausen instances that share their grids (k and
sigma free: the config-4 sweep, multi-start) together.  Controllers of all
instances live in HBM as rows of two [B, d] matrices; every device call of a
tick runs each kernel ONCE over (instance, point) -- csrc/ucp_batch.cuh --
so small grids that leave the GPU idle one instance at a time fill it as a
batch.

Each instance keeps its own round schedule (reference solver.py:234-290:
N_L local iterations, objective, N_P exhaustion iterations, objective,
adaptive split, termination).  Because N_L + N_P = iters_per_round for every
round, all instances reach a round end on the same tick: the host reads the
objectives and decides once per round, and between decisions queues whole
runs of ticks without synchronising.  Instances in a local block and
instances in an exhaustion block run concurrently on two streams ("lanes").

Every instance's controllers, objectives and round reports are bitwise those
of ``solve`` on that instance alone (tests/test_gpu_batch.py).  A numeric
failure in any instance is re-raised exactly by re-running that instance
through ``solve``.
"""
from __future__ import annotations

import ctypes
import threading
import time

import numpy as np
import torch

from . import _lib
from ._device import F64, I64, ptr, to_device_f64
from .device_problem import NO_ERROR
from .grids import ControllerSet, SampledController
from .solver import RoundReport, SolveResult, SolverConfig, adaptive_allocation, solve

__all__ = ["solve_batch", "schedule_rounds", "MAX_BATCH"]

MAX_BATCH = 1024
LAST_STATS: dict = {}  # host-side timing of the last solve_batch (diagnostics)
c_i64, c_dbl, c_vp, c_int, c_i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int, ctypes.c_int32


class WcBatchDesc(ctypes.Structure):
    """struct ucp_wc_batch_desc"""

    _fields_ = [("instances", c_i64), ("a0", c_dbl), ("h0", c_dbl), ("d0", c_i64), ("a1", c_dbl), ("h1", c_dbl),
                ("d1", c_i64), ("y0", c_vp), ("y1", c_vp), ("u0", c_vp), ("u1", c_vp), ("ld0", c_i64),
                ("ld1", c_i64), ("f0", c_vp), ("fw0", c_vp), ("k", c_vp), ("lp0", _lib.LocalParams),
                ("lp1", _lib.LocalParams), ("win_lo0", c_vp), ("win_hi0", c_vp), ("win_lo1", c_vp),
                ("win_hi1", c_vp), ("cand_bound0", c_i64)]


_SIGS = {
    "ucp_wc_batch_create": (c_int, [ctypes.POINTER(WcBatchDesc), ctypes.POINTER(c_vp)]),
    "ucp_wc_batch_destroy": (c_int, [c_vp]),
    "ucp_wc_batch_iterate": (c_int, [c_vp, c_int, c_int, ctypes.POINTER(c_i32), c_i32, c_int, c_vp, c_vp]),
    "ucp_wc_batch_objective": (c_int, [c_vp, c_int, ctypes.POINTER(c_i32), c_i32, c_vp, c_vp, c_vp]),
}
_lib.SIGNATURES.update(_SIGS)


def _bind():
    lib = _lib.load()
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


def _ids(lst):
    return (c_i32 * len(lst))(*lst)


def batchable(problems) -> bool:
    """Witsenhausen instances on identical grids (what the batch engine takes)."""
    from .witsenhausen import Witsenhausen

    if len(problems) < 2 or len(problems) > MAX_BATCH:
        return False
    if not all(type(p) is Witsenhausen and p.arithmetic == "reference" for p in problems):
        return False  # (the batched engine runs the reference's arithmetic only)
    g = problems[0].grids
    return all(p.grids == g for p in problems[1:])


class _Engine:
    """A created ucp_wc_batch plus the HBM rows it points at, reused by every
    solve_batch call of the same shape (no allocation or device sync per call)."""

    def __init__(self, dev, B, g0, g1, cfg, lib):
        from ._device import to_device_i64
        from .grids import node_window_bounds

        self.lib = lib
        d0, d1 = g0.d, g1.d
        ld0, ld1 = d0 + (d0 & 1), d1 + (d1 & 1)
        self.y0, self.y1 = to_device_f64(g0.points, dev), to_device_f64(g1.points, dev)
        self.U0 = torch.zeros((B, ld0), dtype=F64, device=dev)
        self.U1 = torch.zeros((B, ld1), dtype=F64, device=dev)
        self.F0 = torch.zeros((B, ld0), dtype=F64, device=dev)
        self.FW0 = torch.zeros((B, ld0), dtype=F64, device=dev)
        self.K = torch.zeros(B, dtype=F64, device=dev)
        lo0, hi0 = node_window_bounds(g0, cfg.radius_for(g0))
        lo1, hi1 = node_window_bounds(g1, cfg.radius_for(g1))
        self.win = [to_device_i64(x, dev) for x in (lo0, hi0, lo1, hi1)]
        bound0 = int((hi0 - lo0 + 1).sum())
        self.desc = WcBatchDesc(B, g0.a, g0.spacing, d0, g1.a, g1.spacing, d1, ptr(self.y0), ptr(self.y1),
                                ptr(self.U0), ptr(self.U1), ld0, ld1, ptr(self.F0), ptr(self.FW0), ptr(self.K),
                                _lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g0)),
                                _lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g1)),
                                *(ptr(w) for w in self.win), bound0)
        self.handle = c_vp()
        _lib.check(lib.ucp_wc_batch_create(ctypes.byref(self.desc), ctypes.byref(self.handle)), "ucp_wc_batch_create")
        self.err = torch.empty((B, 6), dtype=I64, device=dev)
        self.err_obj = torch.empty(B, dtype=I64, device=dev)
        self.J = torch.zeros((3, B), dtype=F64, device=dev)
        self.lanes = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

    def __del__(self):
        try:
            if self.handle:
                self.lib.ucp_wc_batch_destroy(self.handle)  # synchronises under the capture lock
        except Exception:  # interpreter shutdown
            pass


_ENGINES: dict = {}


def _engine(dev, B, g0, g1, cfg, lib) -> _Engine:
    key = (dev.index, B, g0, g1, cfg.radius_for(g0), cfg.radius_for(g1), cfg.fd_step, cfg.curvature_min,
           cfg.grad_step, cfg.cap_for(g0), cfg.cap_for(g1))
    eng = _ENGINES.get(key)
    if eng is None:
        while len(_ENGINES) >= 2:  # keep the two most recent shapes
            _ENGINES.pop(next(iter(_ENGINES)))
        eng = _ENGINES[key] = _Engine(dev, B, g0, g1, cfg, lib)
    return eng


def schedule_rounds(dev, B: int, cfg: SolverConfig, stats: dict | None = None):
    """Per-instance round schedules of B instances advanced in lock-step ticks
    (reference solver.py:234-290 for each instance).

    ``dev`` provides iterate(kind, ids, iters) [kind 0 local / 1 exhaustion],
    objective(lane, ids, row) [row 0 start, 1 after local, 2 after
    exhaustion], order() [join the two lanes], read() -> (J[3, B], err[B, 6],
    err_obj[B]) after a synchronisation, and failed(i) [raise instance i's
    error].  Returns (final objectives, round reports, terminations).
    Host-side only, so it is tested on CPU with an oracle-backed ``dev``.
    """
    stats = stats if stats is not None else {}
    stats.setdefault("events", 0)
    stats.setdefault("decisions", 0)
    n = cfg.iters_per_round
    adaptive = cfg.fixed_local_iters is None
    everyone = list(range(B))
    dev.objective(0, everyone, 0)
    host_j, _, eo = dev.read()
    bad = (np.asarray(eo) != NO_ERROR).nonzero()[0]
    if bad.size:
        dev.failed(int(bad[0]))
    current = [float(host_j[0, i]) for i in everyone]
    n_local = [n // 2 if adaptive else cfg.fixed_local_iters] * B
    phase = [0] * B  # 0 local block, 1 exhaustion block
    rem = list(n_local)
    round_index = [1] * B
    reports = [[] for _ in range(B)]
    termination = ["max_rounds"] * B
    active = list(everyone)
    t_round = time.perf_counter()
    while active:
        L = [i for i in active if phase[i] == 0]
        E = [i for i in active if phase[i] == 1]
        k = min(rem[i] for i in active)
        if L:
            dev.iterate(0, L, k)
        if E:
            dev.iterate(1, E, k)
        for i in active:
            rem[i] -= k
        ended_l = [i for i in L if rem[i] == 0]
        ended_e = [i for i in E if rem[i] == 0]
        if ended_l:
            dev.objective(0, ended_l, 1)
            for i in ended_l:
                phase[i], rem[i] = 1, n - n_local[i]
        if ended_e:
            dev.objective(1, ended_e, 2)
        dev.order()
        stats["events"] += 1
        if not ended_e:
            continue
        # N_L + N_P = iters_per_round: every active instance ends its round here
        stats["decisions"] += 1
        host_j, e_host, eo_host = dev.read()
        wall = (time.perf_counter() - t_round) * 1000.0
        t_round = time.perf_counter()
        for i in ended_e:
            if (np.asarray(e_host[i]) != NO_ERROR).any() or eo_host[i] != NO_ERROR:
                dev.failed(i)
            after_local, after_exh = float(host_j[1, i]), float(host_j[2, i])
            local_gain = abs(current[i] - after_local)
            exhaustion_gain = abs(after_local - after_exh)
            current[i] = after_exh
            reports[i].append(RoundReport(round_index[i], after_exh, local_gain, exhaustion_gain, n_local[i],
                                          n - n_local[i], wall, after_local))
            if local_gain + exhaustion_gain <= cfg.precision:
                termination[i] = "converged"
                active.remove(i)
                continue
            if round_index[i] == cfg.max_rounds:
                active.remove(i)
                continue
            if adaptive:
                n_local[i], _ = adaptive_allocation(local_gain, exhaustion_gain, n)
            round_index[i] += 1
            phase[i], rem[i] = 0, n_local[i]
    return current, reports, termination


_LOCK = threading.Lock()  # engines are shared: one solve_batch at a time


def solve_batch(problems, cfg: SolverConfig | None = None, initials=None) -> list:
    """Solve Witsenhausen instances sharing their grids as one batch (see module doc)."""
    with _LOCK:
        return _solve_batch(problems, cfg, initials)


def _solve_batch(problems, cfg, initials) -> list:
    from ._device import require_cuda

    t_start = time.perf_counter()
    problems = list(problems)
    if not batchable(problems) and not (len(problems) == 1 and batchable(problems * 2)):
        raise ValueError("solve_batch needs 1..1024 Witsenhausen instances on identical grids")
    cfg = cfg if cfg is not None else SolverConfig()
    B = len(problems)
    initials = list(initials) if initials is not None else [None] * B
    lib = _bind()
    dev = require_cuda(problems[0]._device_arg)
    g0, g1 = problems[0].grids
    d0, d1 = g0.d, g1.d
    eng = _engine(dev, B, g0, g1, cfg, lib)
    U0, U1 = eng.U0, eng.U1
    # per-call rows, staged on the host and uploaded in one copy each
    host = np.zeros((3, B, U0.shape[1]))
    host[0, :, :d0] = np.stack([p._f0 for p in problems])
    host[1, :, :d0] = np.stack([p._fw0 for p in problems])
    host[2, :, :d0] = g0.points
    rows1 = np.zeros((B, U1.shape[1]))
    rows1[:, :d1] = g1.points
    on_dev = []
    for i, U in enumerate(initials):
        if U is None:
            continue
        problems[i].check_controllers(U)
        if U[0].on_device or U[1].on_device:
            on_dev.append(i)
        else:
            host[2, i, :d0] = U.values(0)
            rows1[i, :d1] = U.values(1)
    eng.F0.copy_(torch.from_numpy(host[0]))
    eng.FW0.copy_(torch.from_numpy(host[1]))
    U0.copy_(torch.from_numpy(host[2]))
    U1.copy_(torch.from_numpy(rows1))
    for i in on_dev:
        U0[i, :d0] = initials[i].device_values(0, dev)
        U1[i, :d1] = initials[i].device_values(1, dev)
    eng.K.copy_(torch.tensor([p.k for p in problems], dtype=F64))
    handle = eng.handle
    err, err_obj, J, lanes = eng.err, eng.err_obj, eng.J, eng.lanes
    err.fill_(NO_ERROR)
    err_obj.fill_(NO_ERROR)
    for s_ in lanes:
        s_.wait_stream(torch.cuda.current_stream(dev))

    def call(name, *args):
        _lib.check(getattr(lib, name)(*args), name)

    class Dev:
        """The device side of the schedule (see schedule_rounds)."""

        def iterate(self, kind, ids, iters):
            lane = kind  # lane 0: local-update group, lane 1: exhaustion group
            call("ucp_wc_batch_iterate", handle, lane, kind, _ids(ids), len(ids), iters, ptr(err),
                 lanes[lane].cuda_stream)

        def objective(self, lane, ids, row):
            call("ucp_wc_batch_objective", handle, lane, _ids(ids), len(ids), J[row].data_ptr(), ptr(err_obj),
                 lanes[lane].cuda_stream)

        def order(self):  # instances change lanes at block ends
            lanes[1].wait_stream(lanes[0])
            lanes[0].wait_stream(lanes[1])

        def read(self):
            ts = time.perf_counter()
            lanes[0].synchronize()
            stats["t_sync"] += time.perf_counter() - ts
            return J.cpu().numpy(), err.cpu().numpy(), err_obj.cpu().numpy()

        def failed(self, i):  # re-run alone: raises the reference's exact error
            solve(problems[i], cfg, initials[i])
            raise RuntimeError(f"batch instance {i} flagged a numeric error its single solve did not reproduce")

    stats = {"t_setup": time.perf_counter() - t_start, "t_sync": 0.0}
    try:
        current, reports, termination = schedule_rounds(Dev(), B, cfg, stats)
        torch.cuda.current_stream(dev).wait_stream(lanes[0])
        stats["t_loop_end"] = time.perf_counter() - t_start
        LAST_STATS.clear()
        LAST_STATS.update(stats)
        out = []
        for i in range(B):
            U = ControllerSet((SampledController(g0, U0[i, :d0].clone(), _trusted_device=True),
                               SampledController(g1, U1[i, :d1].clone(), _trusted_device=True)))
            out.append(SolveResult(controllers=U, final_objective=current[i], rounds=tuple(reports[i]),
                                   termination=termination[i]))
        return out
    finally:
        torch.cuda.current_stream(dev).wait_stream(lanes[0])
        torch.cuda.current_stream(dev).wait_stream(lanes[1])
