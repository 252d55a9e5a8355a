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
import time

import numpy as np
import torch

from . import _lib
from ._device import F64, I64, ptr, to_device_f64
from .device_problem import NO_ERROR
from .grids import ControllerSet, SampledController
from .solver import RoundReport, SolveResult, SolverConfig, adaptive_allocation, solve

__all__ = ["solve_batch", "MAX_BATCH"]

MAX_BATCH = 1024
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
    if not all(type(p) is Witsenhausen for p in problems):
        return False
    g = problems[0].grids
    return all(p.grids == g for p in problems[1:])


def solve_batch(problems, cfg: SolverConfig | None = None, initials=None) -> list:
    """Solve Witsenhausen instances sharing their grids as one batch (see module doc)."""
    problems = list(problems)
    if not batchable(problems) and not (len(problems) == 1 and batchable(problems * 2)):
        raise ValueError("solve_batch needs 1..1024 Witsenhausen instances on identical grids")
    cfg = cfg if cfg is not None else SolverConfig()
    B = len(problems)
    initials = list(initials) if initials is not None else [None] * B
    lib = _bind()
    p0 = problems[0]
    D = p0.device_context()
    dev = D.device
    g0, g1 = p0.grids
    d0, d1 = g0.d, g1.d
    ld0, ld1 = d0 + (d0 & 1), d1 + (d1 & 1)

    U0 = torch.zeros((B, ld0), dtype=F64, device=dev)
    U1 = torch.zeros((B, ld1), dtype=F64, device=dev)
    F0 = torch.zeros((B, ld0), dtype=F64, device=dev)
    FW0 = torch.zeros((B, ld0), dtype=F64, device=dev)
    for i, p in enumerate(problems):
        U = p.identity_controllers() if initials[i] is None else initials[i]
        p.check_controllers(U)
        U0[i, :d0] = U.device_values(0, dev)
        U1[i, :d1] = U.device_values(1, dev)
        F0[i, :d0] = to_device_f64(p._f0, dev)
        FW0[i, :d0] = to_device_f64(p._fw0, dev)
    K = torch.tensor([p.k for p in problems], dtype=F64, device=dev)
    lo0, hi0 = D.window(p0, 0, cfg.radius_for(g0))
    lo1, hi1 = D.window(p0, 1, cfg.radius_for(g1))
    bound0 = D.candidate_bound(p0, 0, cfg.radius_for(g0), 0, d0)
    desc = WcBatchDesc(B, g0.a, g0.spacing, d0, g1.a, g1.spacing, d1, ptr(D.y0), ptr(D.y1), ptr(U0), ptr(U1), ld0,
                       ld1, ptr(F0), ptr(FW0), ptr(K),
                       _lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g0)),
                       _lib.LocalParams(cfg.fd_step, cfg.curvature_min, cfg.grad_step, cfg.cap_for(g1)),
                       ptr(lo0), ptr(hi0), ptr(lo1), ptr(hi1), bound0)
    handle = c_vp()
    _lib.check(lib.ucp_wc_batch_create(ctypes.byref(desc), ctypes.byref(handle)), "ucp_wc_batch_create")
    err = torch.full((B, 6), NO_ERROR, dtype=I64, device=dev)
    err_obj = torch.full((B,), NO_ERROR, dtype=I64, device=dev)
    J = torch.zeros((3, B), dtype=F64, device=dev)  # rows: start / after local / after exhaustion
    lanes = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    for s in lanes:
        s.wait_stream(torch.cuda.current_stream(dev))

    def call(name, *args):
        _lib.check(getattr(lib, name)(*args), name)

    def objective(lane, ids, row):
        call("ucp_wc_batch_objective", handle, lane, _ids(ids), len(ids), J[row].data_ptr(), ptr(err_obj),
             lanes[lane].cuda_stream)

    def failed(i):  # re-run alone: raises the reference's exact error
        solve(problems[i], cfg, initials[i])
        raise RuntimeError(f"batch instance {i} flagged a numeric error its single solve did not reproduce")

    try:
        n = cfg.iters_per_round
        adaptive = cfg.fixed_local_iters is None
        everyone = list(range(B))
        objective(0, everyone, 0)
        lanes[0].synchronize()
        host_j = J[0].cpu().numpy()
        bad = (err_obj.cpu().numpy() != NO_ERROR).nonzero()[0]
        if bad.size:
            failed(int(bad[0]))
        current = host_j.astype(np.float64).tolist()
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
                call("ucp_wc_batch_iterate", handle, 0, 0, _ids(L), len(L), k, ptr(err), lanes[0].cuda_stream)
            if E:
                call("ucp_wc_batch_iterate", handle, 1, 1, _ids(E), len(E), k, ptr(err), lanes[1].cuda_stream)
            for i in active:
                rem[i] -= k
            ended_l = [i for i in L if rem[i] == 0]
            ended_e = [i for i in E if rem[i] == 0]
            if ended_l:
                objective(0, ended_l, 1)
                for i in ended_l:
                    phase[i], rem[i] = 1, n - n_local[i]
            if ended_e:
                objective(1, ended_e, 2)
            # instances change lanes at block ends: order the two streams
            lanes[1].wait_stream(lanes[0])
            lanes[0].wait_stream(lanes[1])
            if not ended_e:
                continue
            lanes[0].synchronize()
            host_j = J.cpu().numpy()
            e_host = err.cpu().numpy()
            eo_host = err_obj.cpu().numpy()
            wall = (time.perf_counter() - t_round) * 1000.0
            t_round = time.perf_counter()
            for i in ended_e:
                if (e_host[i] != NO_ERROR).any() or eo_host[i] != NO_ERROR:
                    failed(i)
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
        torch.cuda.current_stream(dev).wait_stream(lanes[0])
        out = []
        for i in everyone:
            U = ControllerSet((SampledController(g0, U0[i, :d0].clone(), _trusted_device=True),
                               SampledController(g1, U1[i, :d1].clone(), _trusted_device=True)))
            out.append(SolveResult(controllers=U, final_objective=current[i], rounds=tuple(reports[i]),
                                   termination=termination[i]))
        return out
    finally:
        lib.ucp_wc_batch_destroy(handle)  # synchronises the device under the capture lock
