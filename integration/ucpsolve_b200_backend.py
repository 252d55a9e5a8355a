"""The `b200` kernel backend a maintainer would add to the reference package
(ucpsolve/kernels.py selects its backend from UCPSOLVE_BACKEND at import,
kernels.py:65-83, 618-637): the same four functions as the numba backend,
NumPy arrays in and out, bound to libucp_b200.so with ctypes and the CUDA
runtime only -- no PyTorch.  INTEGRATION.md, option B.

    import ucpsolve_b200_backend as kb
    t0, t1, t2 = kb.gauss_moments_grid(s, v, a, h, d)      # kernels.py:406-445
    m0, m1, m2 = kb.gauss_moments_points(y, x, w, a, h, d)  # kernels.py:447-486
    J = kb.trapezoid_sum(samples, spacing)                   # kernels.py:136-144
    idx = kb.segmented_argmin(costs, offsets)                # kernels.py:147-160

Every result is bitwise the numba backend's (tests/test_gpu_integration.py
replays the reference's golden vectors through this module).
"""
from __future__ import annotations

import ctypes
import ctypes.util
import os
from pathlib import Path

import numpy as np

_vp, _i64, _d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
_H2D, _D2H = 1, 2
_LIB_PATH = Path(os.environ.get("UCP_B200_LIB", Path(__file__).resolve().parents[1] / "paper_1908_04489_b200" / "libucp_b200.so"))


def _load_cudart():
    for name in ("libcudart.so.12", "libcudart.so", ctypes.util.find_library("cudart")):
        if not name:
            continue
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    import glob
    import sys

    for cand in glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "cuda_runtime", "lib",
                                       "libcudart.so*")):
        return ctypes.CDLL(cand)
    raise OSError("libcudart not found")


_rt = _load_cudart()
_rt.cudaMalloc.argtypes = [ctypes.POINTER(_vp), ctypes.c_size_t]
_rt.cudaFree.argtypes = [_vp]
_rt.cudaMemcpy.argtypes = [_vp, _vp, ctypes.c_size_t, ctypes.c_int]
_rt.cudaDeviceSynchronize.argtypes = []
_lib = ctypes.CDLL(str(_LIB_PATH))
_lib.ucp_last_error.restype = ctypes.c_char_p
_lib.ucp_gauss_moments_grid.argtypes = [_vp, _i64, _vp, _d, _d, _i64, _vp, _vp, _vp, _vp]
_lib.ucp_gauss_moments_points.argtypes = [_vp, _i64, _vp, _vp, _i64, _d, _d, _i64, _vp, _vp, _vp, _vp, _vp]
_lib.ucp_trapezoid_sum.argtypes = [_vp, _i64, _d, _vp, _vp, _vp]
_lib.ucp_segmented_argmin.argtypes = [_vp, _vp, _i64, _vp, _vp]
_lib.ucp_workspace_create.argtypes = [ctypes.POINTER(_vp)]
_WS = _vp()
if _lib.ucp_workspace_create(ctypes.byref(_WS)):
    raise RuntimeError(_lib.ucp_last_error().decode())


def _check(rc, what):
    if rc:
        raise (ValueError if rc == 1 else RuntimeError)(f"{what}: {_lib.ucp_last_error().decode()}")


def _cuda(rc, what):
    if rc:
        raise RuntimeError(f"{what} failed (CUDA error {rc})")


class _Dev:
    """A device buffer holding a copy of a host array (or `nbytes` of scratch)."""

    def __init__(self, host=None, nbytes=0):
        self.nbytes = max(int(host.nbytes if host is not None else nbytes), 8)
        self.p = _vp()
        _cuda(_rt.cudaMalloc(ctypes.byref(self.p), self.nbytes), "cudaMalloc")
        if host is not None and host.nbytes:
            _cuda(_rt.cudaMemcpy(self.p, host.ctypes.data_as(_vp), host.nbytes, _H2D), "cudaMemcpy")

    def to_host(self, dtype, n):
        out = np.empty(n, dtype=dtype)
        if n:
            _cuda(_rt.cudaMemcpy(out.ctypes.data_as(_vp), self.p, out.nbytes, _D2H), "cudaMemcpy")
        return out

    def __del__(self):
        if getattr(self, "p", None):
            _rt.cudaFree(self.p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def gauss_moments_grid(s, v, a, h, d):
    s, v = _f64(s), _f64(v)
    ds, dv = _Dev(s), _Dev(v)
    outs = [_Dev(nbytes=s.nbytes) for _ in range(3)]
    _check(_lib.ucp_gauss_moments_grid(ds.p, s.size, dv.p, float(a), float(h), int(d), *(o.p for o in outs), None),
           "ucp_gauss_moments_grid")
    return tuple(o.to_host(np.float64, s.size) for o in outs)


def gauss_moments_points(y, x, w, a, h, d):
    y, x, w = _f64(y), _f64(x), _f64(w)
    dy, dx, dw = _Dev(y), _Dev(x), _Dev(w)
    outs = [_Dev(nbytes=y.nbytes) for _ in range(3)]
    _check(_lib.ucp_gauss_moments_points(dy.p, y.size, dx.p, dw.p, x.size, float(a), float(h), int(d),
                                         *(o.p for o in outs), _WS, None), "ucp_gauss_moments_points")
    return tuple(o.to_host(np.float64, y.size) for o in outs)


def trapezoid_sum(samples, spacing):
    x = _f64(samples)
    dx, out = _Dev(x), _Dev(nbytes=8)
    _check(_lib.ucp_trapezoid_sum(dx.p, x.size, float(spacing), out.p, None, None), "ucp_trapezoid_sum")
    return float(out.to_host(np.float64, 1)[0])


def segmented_argmin(costs, offsets):
    c = _f64(costs)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    nseg = o.size - 1
    dc, do, out = _Dev(c), _Dev(o), _Dev(nbytes=8 * max(nseg, 1))
    _check(_lib.ucp_segmented_argmin(dc.p, do.p, nseg, out.p, None), "ucp_segmented_argmin")
    return out.to_host(np.int64, nseg)
