"""Monte-Carlo objective on the device.

Two estimators, both evaluating every simulated run in the CUDA kernels of
csrc/ucp_mc.cuh:

* :func:`monte_carlo_objective` -- the reference's own estimator
  (oracle.py:98-105): the draws come from NumPy's seeded PCG64 generator on
  the host in exactly the order ``simulate_cost`` consumes them
  (witsenhausen.py:81-89, zero_delay.py:88-94, inventory.py:152-166), the
  per-sample costs are computed on the device, and mean / standard error are
  NumPy's.  The result is bitwise the reference's for the same seed.
* :func:`device_monte_carlo_objective` -- draws made on the device by a
  counter-based Philox4x32-10 generator, costs and a fixed-order reduction in
  HBM; the samples shard over ranks with one all-gather of chunk partials per
  pass, and the estimate is bitwise independent of the rank count.  This is
  the independent J check at fine grids and large sample counts.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from ._device import F64, ptr
from .distributed import LOCAL, Sharding

__all__ = ["MC_CHUNK", "simulate_cost", "monte_carlo_objective", "device_monte_carlo_objective", "philox_draws"]

MC_CHUNK = 4096  # UCP_MC_CHUNK
MAX_STAGES = 16
KINDS = {"witsenhausen": 0, "zero_delay": 1, "inventory": 2}

c_i32, c_i64, c_u64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class McProblemC(ctypes.Structure):
    """struct ucp_mc_problem"""

    _fields_ = [("kind", c_i32), ("stages", c_i32), ("k", c_dbl), ("sigma", c_dbl), ("power_weight", c_dbl),
                ("quadratic", c_i32), ("reserved", c_i32), ("order_cost", c_dbl), ("holding_rate", c_dbl),
                ("backlog_rate", c_dbl), ("a", c_dbl * MAX_STAGES), ("h", c_dbl * MAX_STAGES),
                ("d", c_i64 * MAX_STAGES), ("pts", c_vp * MAX_STAGES), ("u", c_vp * MAX_STAGES)]


_PP = ctypes.POINTER(McProblemC)
_SIGS = {
    "ucp_mc_streams": (ctypes.c_int, [_PP]),
    "ucp_mc_costs": (ctypes.c_int, [_PP, c_vp, c_i64, c_vp, c_vp]),
    "ucp_mc_philox_draws": (ctypes.c_int, [_PP, c_u64, c_i64, c_i64, c_vp, c_vp]),
    "ucp_mc_partials": (ctypes.c_int, [_PP, c_u64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "ucp_mc_reduce": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
}
_lib.SIGNATURES.update(_SIGS)


def _bind():
    lib = _lib.load()
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


def _kind(problem) -> int:
    try:
        return KINDS[problem.name]
    except KeyError:
        raise TypeError(f"no device Monte-Carlo model for problem {problem.name!r}") from None


def _struct(problem, U):
    """(ucp_mc_problem, device tensors it points to, device, stream)."""
    _bind()
    problem.check_controllers(U)
    D = problem.device_context()
    dev = D.device
    P = McProblemC()
    P.kind = _kind(problem)
    P.stages = problem.M
    keep = []
    if P.kind == 0:
        P.k, P.sigma = problem.k, problem.sigma
    elif P.kind == 1:
        P.power_weight = problem.power_weight
    else:
        P.quadratic = 1 if problem.stage_cost == "quadratic" else 0
        P.order_cost, P.holding_rate, P.backlog_rate = problem.order_cost, problem.holding_rate, problem.backlog_rate
        pts = problem._t  # device grid points (config5.Inventory._build_structs)
        for m in range(problem.M):
            P.pts[m] = ptr(pts[m])
    for m, g in enumerate(problem.grids):
        u = U.device_values(m, dev)
        keep.append(u)
        P.a[m], P.h[m], P.d[m], P.u[m] = g.a, g.spacing, g.d, ptr(u)
    return P, keep, dev, D.stream


def _host_draws(problem, rng, n: int) -> list:
    """The generator calls of the reference's simulate_cost, in its order."""
    kind = _kind(problem)
    if kind == 0:  # witsenhausen.py:83, 86
        return [rng.normal(0.0, problem.sigma, n), rng.normal(0.0, 1.0, n)]
    if kind == 1:  # zero_delay.py:89, 91 (numerics.sample of Uniform(-1, 1))
        return [rng.normal(0.0, 1.0, n), rng.uniform(-1.0, 1.0, n)]
    return [rng.uniform(-1.0, 1.0, n) for _ in range(problem.M + 1)]  # inventory.py:158, 162


def simulate_cost(problem, U, rng, n: int) -> np.ndarray:
    """Per-sample cost of ``n`` simulated runs (the problems' ``simulate_cost``):
    host draws from ``rng`` in the reference's order, costs on the device."""
    n = int(n)
    draws = np.stack(_host_draws(problem, rng, n)) if n > 0 else np.empty((0, 0))
    P, keep, dev, stream = _struct(problem, U)
    if n == 0:
        return np.empty(0)
    d_draws = torch.from_numpy(np.ascontiguousarray(draws)).to(dev)
    out = torch.empty(n, dtype=F64, device=dev)
    _lib.call("ucp_mc_costs", ctypes.byref(P), ptr(d_draws), n, ptr(out), stream)
    return out.cpu().numpy()


def monte_carlo_objective(problem, U, oc):
    """Sample-mean objective and standard error (reference oracle.py:98-105),
    bitwise the reference's for the same ``oc.seed``."""
    problem.check_controllers(U)
    rng = np.random.default_rng(oc.seed)
    costs = simulate_cost(problem, U, rng, oc.mc_samples)
    estimate = float(np.mean(costs))
    stderr = float(np.std(costs, ddof=1) / math.sqrt(oc.mc_samples))
    return estimate, stderr


def philox_draws(problem, U, seed: int, begin: int, end: int) -> np.ndarray:
    """The device generator's draws for samples [begin, end), shape [S, end-begin]
    (test / inspection hook)."""
    P, keep, dev, stream = _struct(problem, U)
    S = _lib.load().ucp_mc_streams(ctypes.byref(P))
    out = torch.empty((S, max(end - begin, 0)), dtype=F64, device=dev)
    _lib.call("ucp_mc_philox_draws", ctypes.byref(P), int(seed) & (2**64 - 1), begin, end, ptr(out), stream)
    return out.cpu().numpy()


def device_monte_carlo_objective(problem, U, n_samples: int, seed: int = 0, sharding: Sharding = LOCAL,
                                 return_device: bool = False):
    """(estimate, stderr) of J over ``n_samples`` device-generated runs.

    Chunks of MC_CHUNK samples are split over the ranks of ``sharding``; each
    pass all-gathers the chunk partials and every rank folds them in the same
    order, so all ranks (and every world size) get the same bits.  Two passes:
    the mean, then the squared deviations (np.std's two-pass form).
    """
    n = int(n_samples)
    if n < 1:
        raise ValueError(f"mc_samples must be a positive integer (got {n_samples})")
    P, keep, dev, stream = _struct(problem, U)
    seed = int(seed) & (2**64 - 1)
    chunks = -(-n // MC_CHUNK)
    cb, ce = sharding.bounds(chunks)
    buf = sharding.out_buffer(chunks, dev)
    sums = torch.empty(2, dtype=F64, device=dev)
    for p in range(2):
        _lib.call("ucp_mc_partials", ctypes.byref(P), seed, n, cb, ce, None if p == 0 else ptr(sums),
                  buf.data_ptr() + 8 * cb, stream)
        sharding.allgather_(buf)
        _lib.call("ucp_mc_reduce", ptr(buf), chunks, sums.data_ptr() + 8 * p, stream)
    if return_device:
        return sums
    total, sq = (float(v) for v in sums.cpu().numpy())
    estimate = total / n
    stderr = math.sqrt(sq / (n - 1)) / math.sqrt(n) if n > 1 else math.nan
    return estimate, stderr
