"""ctypes binding of the C ABI in include/ucp_b200.h (libucp_b200.so).

This is the host side of the drop-in boundary.  There is no CPU fallback:
importing the binding without the built library, or calling into it without
a CUDA device, raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("UCP_B200_LIB", PKG / "libucp_b200.so"))

UCP_OK = 0
UCP_ERR_ARG = 1
UCP_ERR_CUDA = 3
NO_ERROR = (1 << 63) - 1  # UCP_NO_ERROR
ABI_VERSION = 3  # UCP_ABI_VERSION (3: ucp_wc_problem.flags)
WC_FAST = 1  # UCP_WC_FAST
WC_TABLE = 2  # UCP_WC_TABLE

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_int = ctypes.c_int


class WcProblem(ctypes.Structure):
    """struct ucp_wc_problem"""

    _fields_ = [
        ("k", c_dbl),
        ("a0", c_dbl), ("h0", c_dbl), ("d0", c_i64),
        ("a1", c_dbl), ("h1", c_dbl), ("d1", c_i64),
        ("y0", c_vp), ("y1", c_vp), ("f0", c_vp), ("fw0", c_vp),
        ("flags", c_i64),
    ]


class LocalParams(ctypes.Structure):
    """struct ucp_local_params"""

    _fields_ = [("fd_step", c_dbl), ("curvature_min", c_dbl), ("grad_step", c_dbl),
                ("newton_cap", c_dbl)]


# name -> (restype, argtypes); mirrors include/ucp_b200.h one to one
SIGNATURES = {
    "ucp_abi_version": (c_int, []),
    "ucp_status_string": (ctypes.c_char_p, [c_int]),
    "ucp_last_error": (ctypes.c_char_p, []),
    "ucp_launch_count": (c_i64, []),
    "ucp_workspace_create": (c_int, [ctypes.POINTER(c_vp)]),
    "ucp_workspace_destroy": (c_int, [c_vp]),
    "ucp_workspace_recycle": (c_int, [c_vp]),
    "ucp_workspace_reserve": (c_int, [c_vp, c_i64, c_i64, c_i64]),
    "ucp_gauss_moments_grid": (c_int, [c_vp, c_i64, c_vp, c_dbl, c_dbl, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ucp_gauss_moments_points": (c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_i64, c_vp, c_vp,
                                         c_vp, c_vp, c_vp]),
    "ucp_trapezoid_sum": (c_int, [c_vp, c_i64, c_dbl, c_vp, c_vp, c_vp]),
    "ucp_segmented_argmin": (c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "ucp_device_libm": (c_int, [c_int, c_vp, c_i64, c_vp, c_vp]),
    "ucp_flatten_windows": (c_int, [c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ucp_wc_stage0_cost": (c_int, [ctypes.POINTER(WcProblem), c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                   c_vp, c_vp]),
    "ucp_wc_stage0_cost_ws": (c_int, [ctypes.POINTER(WcProblem), c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                      c_vp, c_vp, c_vp]),
    "ucp_wc_stage1_cost": (c_int, [ctypes.POINTER(WcProblem), c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp,
                                   c_vp, c_vp]),
    "ucp_wc_local_update": (c_int, [ctypes.POINTER(WcProblem), c_int, c_vp, c_vp, ctypes.POINTER(LocalParams),
                                    c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "ucp_wc_exhaustion": (c_int, [ctypes.POINTER(WcProblem), c_int, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64,
                                  c_vp, c_vp, c_vp, c_vp]),
    "ucp_wc_run_block": (c_int, [ctypes.POINTER(WcProblem), c_int, c_int, c_vp, c_vp, ctypes.POINTER(LocalParams),
                                 c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ucp_wc_run_block_graph": (c_int, [ctypes.POINTER(WcProblem), c_int, c_int, c_vp, c_vp,
                                       ctypes.POINTER(LocalParams), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                       c_vp, c_vp]),
    "ucp_wc_objective_terms": (c_int, [ctypes.POINTER(WcProblem), c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                                       c_vp]),
    "ucp_wc_objective_terms_ws": (c_int, [ctypes.POINTER(WcProblem), c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                                          c_vp, c_vp]),
    "ucp_fp64_probe": (c_int, [c_int, c_int, c_int, c_vp, c_vp]),
    "ucp_walk_node_counter": (c_int, [c_vp]),
}


class UcpError(RuntimeError):
    """A CUDA-level failure inside libucp_b200 (status UCP_ERR_CUDA)."""


_LIB = None


def load() -> ctypes.CDLL:
    """Load libucp_b200.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ucp_abi_version() != ABI_VERSION:
        raise ImportError(f"libucp_b200 ABI {lib.ucp_abi_version()} != {ABI_VERSION}")
    _LIB = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == UCP_OK:
        return
    msg = load().ucp_last_error().decode(errors="replace")
    if rc == UCP_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    raise UcpError(f"{what}: {msg} (status {rc})")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().ucp_launch_count())
