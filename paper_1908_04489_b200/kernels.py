"""Drop-in for the reference's ``kernels`` module (kernels.py:31-45, 618-658).

Same function names and signatures as the numba backend; inputs may be NumPy
arrays (copied to the device and back, like a plugin call) or float64 CUDA
tensors (then the results stay on the device).  Every call runs a
libucp_b200 kernel -- there is no NumPy or CPU fallback.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib
from ._device import F64, I64, ptr, require_cuda, stream_ptr, to_device_f64, to_device_i64

__all__ = [
    "BACKEND",
    "NUMBA_ENABLED",
    "GAUSS_CUT",
    "set_workers",
    "max_workers",
    "trapezoid_sum",
    "flatten_windows",
    "segmented_argmin",
    "gauss_moments_grid",
    "gauss_moments_points",
    "unif_moments_grid",
    "unif_ball_sum",
    "unif_propagate",
    "unif_moments_points",
    "implementations",
    "device_libm",
]

BACKEND = "b200"
# No numba here; every kernel follows the numba backend's semantics (bitwise its
# results, flatten_windows' dedup included), which is what the reference's tests
# gate on NUMBA_ENABLED -- NUMBA_SEMANTICS says so without claiming numba.
NUMBA_ENABLED = False
NUMBA_SEMANTICS = True
GAUSS_CUT = 12.0
_TLS = threading.local()  # one scratch workspace per (host thread, device)


def max_workers() -> int:
    """One process drives one GPU; multi-GPU runs shard across processes."""
    return 1


def set_workers(n: int) -> int:
    if n < 1:
        raise ValueError(f"workers must be at least 1 (got {n})")
    return 1


def _device_of(*xs):
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device, True
    return require_cuda(), False


def _workspace(device):
    cache = getattr(_TLS, "ws", None)
    if cache is None:
        cache = _TLS.ws = {}
    if device.index not in cache:
        ws = ctypes.c_void_p()
        _lib.call("ucp_workspace_create", ctypes.byref(ws))
        cache[device.index] = ws
    return cache[device.index]


def _out(t, keep):
    return t if keep else t.cpu().numpy()


def gauss_moments_grid(s, v, a, h, d):
    """T0, T1, T2 at centres s (kernels.py:406-445)."""
    dev, keep = _device_of(s, v)
    sd, vd = to_device_f64(s, dev), to_device_f64(v, dev)
    n = sd.numel()
    outs = [torch.empty(n, dtype=F64, device=dev) for _ in range(3)]
    _lib.call("ucp_gauss_moments_grid", ptr(sd), n, ptr(vd), float(a), float(h), int(d),
              *(ptr(o) for o in outs), stream_ptr(dev))
    return tuple(_out(o, keep) for o in outs)


def gauss_moments_points(y, x, w, a, h, d):
    """Moments over scattered support points (kernels.py:447-486)."""
    dev, keep = _device_of(y, x, w)
    yd, xd, wd = to_device_f64(y, dev), to_device_f64(x, dev), to_device_f64(w, dev)
    n = yd.numel()
    outs = [torch.empty(n, dtype=F64, device=dev) for _ in range(3)]
    _lib.call("ucp_gauss_moments_points", ptr(yd), n, ptr(xd), ptr(wd), xd.numel(), float(a), float(h),
              int(d), *(ptr(o) for o in outs), _workspace(dev), stream_ptr(dev))
    return tuple(_out(o, keep) for o in outs)


def trapezoid_sum(samples, spacing):
    """Serial ascending trapezoid on the device (kernels.py:136-144)."""
    dev, _ = _device_of(samples)
    sd = to_device_f64(samples, dev)
    out = torch.empty(1, dtype=F64, device=dev)
    _lib.call("ucp_trapezoid_sum", ptr(sd), sd.numel(), float(spacing), ptr(out), None, stream_ptr(dev))
    return float(out.item())


def segmented_argmin(costs, offsets):
    """First index of the strict minimum per segment (kernels.py:147-160)."""
    dev, keep = _device_of(costs, offsets)
    cd, od = to_device_f64(costs, dev), to_device_i64(offsets, dev)
    nseg = od.numel() - 1
    out = torch.empty(max(nseg, 1), dtype=I64, device=dev)
    _lib.call("ucp_segmented_argmin", ptr(cd), ptr(od), nseg, ptr(out), stream_ptr(dev))
    out = out[:nseg]
    return out if keep else out.cpu().numpy()


def flatten_windows(values, lo, hi):
    """Flat candidates and offsets of every window values[lo[i]..hi[i]]
    (kernels.py:163-187, numba variant: a value equal to an earlier one of the
    same window is dropped, window order kept)."""
    dev, keep = _device_of(values, lo, hi)
    vd, lod, hid = to_device_f64(values, dev), to_device_i64(lo, dev), to_device_i64(hi, dev)
    n = lod.numel()
    if hid.numel() != n:
        raise ValueError("lo and hi disagree")
    width = (hid - lod + 1).clamp(min=0)
    if n and bool(((width > 0) & ((lod < 0) | (hid >= vd.numel()))).any()):
        raise ValueError("window bounds outside the values")
    cap = int(width.sum().item()) if n else 0
    flat = torch.empty(max(cap, 1), dtype=F64, device=dev)
    offsets = torch.empty(n + 1, dtype=I64, device=dev)
    _lib.call("ucp_flatten_windows", ptr(vd), vd.numel(), ptr(lod), ptr(hid), n, ptr(flat), ptr(offsets),
              _workspace(dev), stream_ptr(dev))
    total = int(offsets[n].item())
    return _out(flat[:total], keep), _out(offsets, keep)


def _unif(name, n_out, n, *args, dev, keep, length=None):
    from .config5 import _bind

    _bind()
    outs = [torch.empty(max(length if length is not None else n, 1), dtype=F64, device=dev) for _ in range(n_out)]
    _lib.call(name, *args, *(ptr(o) for o in outs), stream_ptr(dev))
    outs = [o[:length if length is not None else n] for o in outs]
    return tuple(_out(o, keep) for o in outs) if n_out > 1 else _out(outs[0], keep)


def unif_moments_grid(x, v, a, h, d, rad):
    """Uniform-noise moments of a clamped step function v at centres x (kernels.py:488-525)."""
    dev, keep = _device_of(x, v)
    xd, vd = to_device_f64(x, dev), to_device_f64(v, dev)
    return _unif("ucp_unif_moments_grid", 3, xd.numel(), ptr(xd), xd.numel(), ptr(vd), float(a), float(h), int(d),
                 float(rad), dev=dev, keep=keep)


def unif_ball_sum(x, g, a, h, d, rad):
    """Ball average of g over [x - rad, x + rad] (kernels.py:528-555)."""
    dev, keep = _device_of(x, g)
    xd, gd = to_device_f64(x, dev), to_device_f64(g, dev)
    return _unif("ucp_unif_ball_sum", 1, xd.numel(), ptr(xd), xd.numel(), ptr(gd), float(a), float(h), int(d),
                 float(rad), dev=dev, keep=keep)


def unif_propagate(masses, centers, a, h, d, rad):
    """Density on the d grid cells of masses spread uniformly around centres (kernels.py:558-577)."""
    dev, keep = _device_of(masses, centers)
    md, cd = to_device_f64(masses, dev), to_device_f64(centers, dev)
    return _unif("ucp_unif_propagate", 1, md.numel(), ptr(md), ptr(cd), md.numel(), float(a), float(h), int(d),
                 float(rad), dev=dev, keep=keep, length=int(d))


def unif_moments_points(y, centers, w, vals, a, h, d, rad):
    """Cell-overlap moments over scattered support points (kernels.py:580-615)."""
    dev, keep = _device_of(y, centers, w, vals)
    yd, cd = to_device_f64(y, dev), to_device_f64(centers, dev)
    wd, vd = to_device_f64(w, dev), to_device_f64(vals, dev)
    return _unif("ucp_unif_moments_points", 3, yd.numel(), ptr(yd), yd.numel(), ptr(cd), ptr(wd), ptr(vd), cd.numel(),
                 float(a), float(h), int(d), float(rad), dev=dev, keep=keep)


def implementations() -> dict:
    """The heavy kernels by name, as ``(device_impl, None)`` (kernels.py:640-658
    returns ``(numba_impl_or_None, numpy_impl)``; this backend has one
    implementation per kernel, bitwise the numba one)."""
    names = ["gauss_moments_grid", "gauss_moments_points", "unif_moments_grid", "unif_ball_sum",
             "unif_propagate", "unif_moments_points"]
    return {name: (globals()[name], None) for name in names}


def device_libm(which: str, x):
    """glibc-exact exp / erf / phi_cdf evaluated on the device (parity tests)."""
    code = {"exp": 0, "erf": 1, "phi_cdf": 2}[which]
    dev, keep = _device_of(x)
    xd = to_device_f64(x, dev)
    out = torch.empty_like(xd)
    _lib.call("ucp_device_libm", code, ptr(xd), xd.numel(), ptr(out), stream_ptr(dev))
    return _out(out, keep)
