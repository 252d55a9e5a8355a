"""The product's glibc-exact exp/erf port (csrc/ucp_libm.h), host build.

The same header is compiled into the CUDA kernels; the GPU test
(test_gpu_parity.py::test_device_libm) repeats the comparison on device.
"""
import ctypes
import subprocess
from pathlib import Path

import pytest

NATIVE = Path(__file__).resolve().parent / "native"


@pytest.fixture(scope="module")
def port():
    subprocess.run(["make", "-s", "-C", str(NATIVE)], check=True)
    L = ctypes.CDLL(str(NATIVE / "_build" / "liblibm_port_check.so"))
    L.compare_uniform.restype = ctypes.c_int64
    L.compare_uniform.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                                  ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    L.compare_core.restype = ctypes.c_int64
    L.compare_core.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                               ctypes.POINTER(ctypes.c_double)]
    L.compare_bits.restype = ctypes.c_int64
    L.compare_bits.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                               ctypes.POINTER(ctypes.c_double)]
    return L


RANGES = [
    (0, -72.5, 0.5),      # stage-0 / stage-1 pdf arguments
    (0, -1e-3, 1e-3),     # recurrence ratios exp(-h*(tt+h/2)), exp(-h*h)
    (0, -37.0, -0.5),     # erf's internal exp(-z*z-0.5625)
    (0, -745.5, 709.9),   # full finite range incl. the specialcase branch
    (0, -1100.0, 1100.0), # overflow / underflow
    (1, -8.5, 8.5),       # phi_cdf arguments z/sqrt(2), |z| < 12
    (1, -1.3, 1.3),
    (1, -1e-8, 1e-8),
]


@pytest.mark.parametrize("which,lo,hi", RANGES)
def test_uniform_ranges_bitwise(port, which, lo, hi):
    first = ctypes.c_double(0.0)
    bad = port.compare_uniform(which, 2_000_000, 1234 + which, lo, hi, ctypes.byref(first))
    assert bad == 0, f"{bad} mismatches, first at {first.value!r}"


@pytest.mark.parametrize("which", [0, 1])
def test_random_bit_patterns(port, which):
    first = ctypes.c_double(0.0)
    bad = port.compare_bits(which, 2_000_000, 99, ctypes.byref(first))
    assert bad == 0, f"{bad} mismatches, first at {first.value!r}"


@pytest.mark.parametrize("lo,hi", [(-72.5, 0.0), (-511.9, 511.9), (-1e-3, 1e-3)])
def test_exp_core_main_path_equivalence(port, lo, hi):
    """The kernels' branch-free exp (main path only) == glibc exp for |x| < 512."""
    first = ctypes.c_double(0.0)
    bad = port.compare_core(3_000_000, 5, lo, hi, ctypes.byref(first))
    assert bad == 0, f"{bad} mismatches, first at {first.value!r}"
