"""Grids and step-function controllers with device-resident values.

Same public surface as the reference's ``grids`` module (grids.py:1-195):
``Grid``, ``SampledController``, ``ControllerSet``, nearest-point snapping and
search windows.  The difference is storage: a controller's value vector may
live in HBM (a float64 CUDA tensor written by a device sweep) and is copied
to the host only when ``.values`` is read, so a solve keeps every controller
on the GPU from start to finish.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Grid",
    "SampledController",
    "ControllerSet",
    "make_grid",
    "init_identity",
    "eval_controller",
    "eval_controller_many",
    "nearest_index",
    "nearest_indices",
    "window_bounds",
    "window_indices",
    "node_window_bounds",
]

# index-unit slack for exact-boundary windows (reference grids.py:31)
WINDOW_FUZZ = 1e-9


@dataclass(frozen=True)
class Grid:
    """``d`` equispaced points over ``[a, b]`` (np.linspace, like the reference)."""

    a: float
    b: float
    d: int
    points: np.ndarray = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        if not (np.isfinite(self.a) and np.isfinite(self.b)):
            raise ValueError(f"grid.a/grid.b must be finite (got a={self.a}, b={self.b})")
        if not self.a < self.b:
            raise ValueError(f"grid.a must be below grid.b (got a={self.a}, b={self.b})")
        if int(self.d) != self.d or self.d < 2:
            raise ValueError(f"grid.d must be an integer of at least 2 (got {self.d})")
        pts = np.linspace(self.a, self.b, self.d)
        pts.setflags(write=False)
        object.__setattr__(self, "points", pts)

    @property
    def spacing(self) -> float:
        return (self.b - self.a) / (self.d - 1)


def make_grid(a: float, b: float, d: int) -> Grid:
    return Grid(float(a), float(b), int(d))


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


_CONTENT_KEYS = itertools.count(1)


def content_key(t) -> int:
    """A nonzero 64-bit key for the CONTENTS of a controller's device tensor
    (0: none): a serial stamped when the controller adopts or creates the
    tensor, combined with the tensor's in-place version counter, so a key is
    never shared by different contents (ucp_inv_problem.ukey)."""
    serial = getattr(t, "_ucp_serial", 0)
    if not serial:
        return 0
    try:
        if t.is_inference():  # no version counter: writes cannot be seen, so no reuse
            return 0
        version = t._version
    except RuntimeError:
        return 0
    if version >= 1 << 20 or serial >= 1 << 43:
        return 0
    return (serial << 20) | version


class SampledController:
    """Immutable step-function controller: one float64 value per grid point.

    ``values`` may be given as a NumPy array (validated like the reference,
    grids.py:76-85) or as a float64 CUDA tensor.  Device tensors produced by
    the solver's sweeps are finite-checked on the device (the sweep's error
    slots), so they are adopted without a host round trip.
    """

    __slots__ = ("grid", "_host", "_dev")

    def __init__(self, grid: Grid, values, *, _trusted_device: bool = False):
        object.__setattr__(self, "grid", grid)
        object.__setattr__(self, "_host", None)
        object.__setattr__(self, "_dev", None)
        if _is_tensor(values) and values.is_cuda:
            import torch

            t = values.detach()
            if t.dtype != torch.float64 or t.dim() != 1 or t.numel() != grid.d:
                raise ValueError(f"controller needs {grid.d} values, got shape {tuple(t.shape)}")
            # a caller's tensor is copied (the reference copies its input too,
            # grids.py:76-85): later writes to it -- including ones the version
            # counter does not see (.data, DLPack, raw pointers) -- can neither
            # change this immutable controller nor a content-keyed cache entry;
            # the library's own sweep outputs are adopted as they are
            t = t.contiguous() if _trusted_device else t.clone(memory_format=torch.contiguous_format)
            if not _trusted_device:
                ok = torch.isfinite(t)
                if not bool(ok.all()):
                    bad = int(torch.nonzero(~ok)[0, 0])
                    raise ValueError(f"controller value at grid point {bad} is not finite")
            t._ucp_serial = next(_CONTENT_KEYS)
            object.__setattr__(self, "_dev", t)
            return
        vals = np.array(values.cpu() if _is_tensor(values) else values, dtype=np.float64)
        if vals.ndim != 1 or vals.size != grid.d:
            raise ValueError(f"controller needs {grid.d} values, got shape {vals.shape}")
        finite = np.isfinite(vals)
        if not finite.all():
            raise ValueError(f"controller value at grid point {int(np.flatnonzero(~finite)[0])} is not finite")
        vals.setflags(write=False)
        object.__setattr__(self, "_host", vals)

    def __setattr__(self, name, value):
        raise AttributeError("SampledController is immutable")

    @property
    def values(self) -> np.ndarray:
        """Host copy of the value vector (read-only; copied once from HBM)."""
        if self._host is None:
            host = self._dev.cpu().numpy()
            host.setflags(write=False)
            object.__setattr__(self, "_host", host)
        return self._host

    def device_values(self, device):
        """The value vector as a float64 CUDA tensor on ``device`` (cached)."""
        import torch

        dev = self._dev
        if dev is None or dev.device != torch.device(device):
            dev = torch.from_numpy(np.array(self.values)).to(device)
            dev._ucp_serial = next(_CONTENT_KEYS)
            object.__setattr__(self, "_dev", dev)
        return dev

    @property
    def on_device(self) -> bool:
        return self._dev is not None

    def with_values(self, values) -> "SampledController":
        return SampledController(self.grid, values)

    def __repr__(self):
        where = "cuda" if self._dev is not None else "host"
        return f"SampledController(grid={self.grid!r}, {where})"


@dataclass(frozen=True)
class ControllerSet:
    """One controller per stage (reference grids.py:92-118)."""

    controllers: tuple

    def __post_init__(self):
        object.__setattr__(self, "controllers", tuple(self.controllers))
        if not self.controllers:
            raise ValueError("controller set must hold at least one stage")

    def __len__(self) -> int:
        return len(self.controllers)

    def __getitem__(self, m: int) -> SampledController:
        return self.controllers[m]

    def values(self, m: int) -> np.ndarray:
        return self.controllers[m].values

    def device_values(self, m: int, device):
        return self.controllers[m].device_values(device)

    def grid(self, m: int) -> Grid:
        return self.controllers[m].grid

    def replace(self, m: int, controller: SampledController) -> "ControllerSet":
        ctrls = list(self.controllers)
        ctrls[m] = controller
        return ControllerSet(tuple(ctrls))


def init_identity(grid: Grid) -> SampledController:
    return SampledController(grid, grid.points.copy())


def nearest_indices(grid: Grid, y) -> np.ndarray:
    """Nearest grid index, exact midpoints rounding down, clamped (grids.py:126-145)."""
    t = (np.asarray(y, dtype=np.float64) - grid.a) / grid.spacing
    return np.clip(np.ceil(t - 0.5).astype(np.int64), 0, grid.d - 1)


def nearest_index(grid: Grid, y: float) -> int:
    return int(nearest_indices(grid, np.array([y]))[0])


def eval_controller(ctrl: SampledController, y: float) -> float:
    return float(ctrl.values[nearest_index(ctrl.grid, y)])


def eval_controller_many(ctrl: SampledController, y) -> np.ndarray:
    return ctrl.values[nearest_indices(ctrl.grid, y)]


def _bounds(grid: Grid, centres, r):
    if not r > 0.0:
        raise ValueError(f"window radius must be positive (got {r})")
    h = grid.spacing
    lo = np.ceil((centres - r - grid.a) / h - WINDOW_FUZZ).astype(np.int64)
    hi = np.floor((centres + r - grid.a) / h + WINDOW_FUZZ).astype(np.int64)
    ic = nearest_indices(grid, centres)
    lo = np.maximum(0, np.minimum(lo, ic))
    hi = np.minimum(grid.d - 1, np.maximum(hi, ic))
    return lo, hi


def window_bounds(grid: Grid, y_center: float, r: float) -> tuple[int, int]:
    """Inclusive bounds of {i : |y_i - y_center| <= r}, always holding the nearest point."""
    lo, hi = _bounds(grid, np.array([float(y_center)]), r)
    return int(lo[0]), int(hi[0])


def window_indices(grid: Grid, y_center: float, r: float) -> range:
    lo, hi = window_bounds(grid, y_center, r)
    return range(lo, hi + 1)


def node_window_bounds(grid: Grid, r: float):
    """Window bounds of every grid point (grids.py:180-195); same arithmetic."""
    return _bounds(grid, grid.points, r)
