"""Device-side plumbing shared by the device problems: the lazy error log
(phase failures are atomically recorded on the GPU and raised at the next
synchronisation point with the reference's exception) and a generic device
context used by the config-5 problems."""
from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np
import torch

from . import _lib
from ._device import I64, ptr, require_cuda, stream_ptr, to_device_i64
from .distributed import Sharding
from .grids import node_window_bounds
from .problem import NumericError

NO_ERROR = _lib.NO_ERROR


class ErrorLog:
    """Device-side failure slots, one row of 3 int64 per phase, read lazily.

    A phase never stalls the stream to look for non-finite values: it
    atomicMin's the first offending grid point into its row, and the host
    reads all pending rows at the next synchronisation point (the objective,
    or the end of the solve).  The first phase (in execution order) with a
    failure raises exactly the exception the reference raises at that phase;
    work issued after it is discarded with the exception.
    """

    def __init__(self, device, problem, capacity: int = 1024):
        self.device = device
        # weak: problem -> context -> log -> problem would be a cycle, and a
        # cycle is only freed by the cyclic GC -- at an arbitrary moment, e.g.
        # inside another solve, where the context's teardown synchronises
        # the device
        self._problem = weakref.ref(problem) if problem is not None else (lambda: None)
        self.rows = torch.full((capacity, 3), NO_ERROR, dtype=I64, device=device)
        self.meta: list[tuple] = []

    @property
    def problem(self):
        return self._problem()

    def slot(self, kind: str, stage: int, sharding: Sharding) -> torch.Tensor:
        if len(self.meta) == self.rows.shape[0]:
            self.flush(sharding)
        row = self.rows[len(self.meta)]
        self.meta.append((kind, stage))
        return row

    def slots(self, metas: list, sharding: Sharding) -> torch.Tensor:
        """Contiguous rows for a run of phases (one native block call)."""
        need = len(metas)
        if len(self.meta) + need > self.rows.shape[0]:
            self.flush(sharding)
            if need > self.rows.shape[0]:
                self.rows = torch.full((need, 3), NO_ERROR, dtype=I64, device=self.device)
        start = len(self.meta)
        self.meta.extend(metas)
        return self.rows[start:start + need]

    def flush(self, sharding: Sharding, extra: torch.Tensor | None = None):
        """Read the pending rows (one device-to-host copy, together with the
        int64 tensor ``extra`` if given, whose host copy is returned) and
        raise the first recorded failure."""
        n = len(self.meta)
        if n == 0:
            return None if extra is None else extra.cpu().numpy()
        rows = self.rows[:n]
        sharding.allreduce_min_(rows)
        if extra is None:
            host = rows.cpu().numpy().copy()  # (a CPU tensor's .cpu() is itself: rows are reset below)
            extra_host = None
        else:
            both = torch.cat([rows.reshape(-1), extra.reshape(-1)]).cpu().numpy()
            host, extra_host = both[: 3 * n].reshape(n, 3), both[3 * n:]
        rows.fill_(NO_ERROR)
        meta, self.meta = self.meta, []
        for entry, row in zip(meta, host):
            kind, m = entry[0], entry[1]
            if not (row != NO_ERROR).any():
                continue
            if kind == "objective":
                # a deferred objective (payload: its controller set); its row
                # sits between the phases queued before and after it
                raise _objective_error(self.problem, entry[2], int(row[0]))
            if kind == "block":
                # a graph-replayed block only records the minimum over its
                # iterations: re-run it eagerly from its input snapshot so the
                # first failing phase raises exactly the reference's error
                self.problem._replay_block_error(entry[2], sharding)
                raise AssertionError("block failure did not reproduce")
            raise _phase_error(self.problem, kind, m, row)
        return extra_host


def _objective_error(problem, U, bad):
    g = problem.grids[0]
    return NumericError(
        f"{problem.name}: non-finite objective integrand at stage 0, grid point {bad} "
        f"(y={g.points[bad]!r}, u={U.values(0)[bad]!r})")


def _phase_error(problem, kind, m, row):
    name = problem.name if problem is not None else "witsenhausen"
    pts = problem.grids[m].points if problem is not None else None
    phase = {"local": "local-update", "exhaustion": "partial-exhaustion"}[kind]
    for slot in range(3 if kind == "local" else 1):
        i = int(row[slot])
        if i == NO_ERROR:
            continue
        if slot == 2:  # grids.py: SampledController rejects non-finite values
            return ValueError(f"controller value at grid point {i} is not finite")
        y = pts[i] if pts is not None else float("nan")
        return NumericError(
            f"{name}: non-finite marginal cost in {phase} phase at stage {m}, grid point {i} (y={y!r})")
    raise AssertionError("no failure in row")




# Released workspaces, per device, for the next problem (ucp_workspace_recycle):
# a fresh problem -- e.g. every solve of a parameter sweep -- reuses grown
# scratch buffers and updates the previous problem's captured block graphs in
# place instead of allocating and instantiating anew.
_POOL: dict = {}
_POOL_LOCK = threading.Lock()
POOL_MAX = 2  # workspaces kept per device


def _pool_take(index: int):
    with _POOL_LOCK:
        free = _POOL.get(index)
        return free.pop() if free else None


def _pool_give(lib, index: int, ws) -> None:
    """Recycle ws into the pool (or destroy it when the pool is full).  Runs
    from __del__, in whatever thread the collector picks: the library takes
    its capture lock for the device synchronisation."""
    with _POOL_LOCK:
        free = _POOL.setdefault(index, [])
        if len(free) < POOL_MAX and lib.ucp_workspace_recycle(ws) == 0:
            free.append(ws)
            return
    lib.ucp_workspace_destroy(ws)


class DeviceContext:
    """Workspace, error log and cached window bounds of one device problem."""

    def __init__(self, prob, device=None):
        self.lib = _lib.load()
        self.device = require_cuda(device)
        ws = _pool_take(self.device.index)
        if ws is None:
            ws = ctypes.c_void_p()
            _lib.call("ucp_workspace_create", ctypes.byref(ws))
        self.ws = ws
        self.errors = ErrorLog(self.device, prob)
        self.windows: dict = {}
        self.plans: dict = {}  # ((stage, radius), world) -> shard bounds (multi-rank sweeps)

    def __del__(self):
        try:
            if self.ws:
                # recycle/destroy synchronise the device themselves, under the
                # library's capture lock (a bare device sync here -- the GC may
                # run this in any thread -- would invalidate another thread's
                # graph capture)
                _pool_give(self.lib, self.device.index, self.ws)
        except Exception:  # interpreter shutdown
            pass

    @property
    def stream(self) -> int:
        return stream_ptr(self.device)

    def window(self, prob, m: int, r: float):
        key = (m, float(r))
        if key not in self.windows:
            lo, hi = node_window_bounds(prob.grids[m], r)
            widths = np.concatenate([[0], np.cumsum(hi - lo + 1)])
            self.windows[key] = (to_device_i64(lo, self.device), to_device_i64(hi, self.device),
                                 int((hi - lo).max()) + 1, widths)
        return self.windows[key][:2]

    def candidate_bound(self, prob, m: int, r: float, begin: int, end: int) -> int:
        """Sum of window widths over [begin, end): an upper bound on the deduped candidates."""
        self.window(prob, m, r)
        widths = self.windows[(m, float(r))][3]
        return int(widths[end] - widths[begin])

    def window_width(self, prob, m: int, r: float) -> int:
        self.window(prob, m, r)
        return self.windows[(m, float(r))][2]
