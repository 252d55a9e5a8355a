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
    "GAUSS_CUT",
    "set_workers",
    "max_workers",
    "trapezoid_sum",
    "segmented_argmin",
    "gauss_moments_grid",
    "gauss_moments_points",
    "device_libm",
]

BACKEND = "b200"
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


def device_libm(which: str, x):
    """glibc-exact exp / erf / phi_cdf evaluated on the device (parity tests)."""
    code = {"exp": 0, "erf": 1, "phi_cdf": 2}[which]
    dev, keep = _device_of(x)
    xd = to_device_f64(x, dev)
    out = torch.empty_like(xd)
    _lib.call("ucp_device_libm", code, ptr(xd), xd.numel(), ptr(out), stream_ptr(dev))
    return _out(out, keep)
