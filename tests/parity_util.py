"""Shared parity assertions for the test-suite."""
import numpy as np


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a = np.atleast_1d(np.asarray(a, dtype=np.float64))
    b = np.atleast_1d(np.asarray(b, dtype=np.float64))
    assert a.shape == b.shape, (what, a.shape, b.shape)
    a, b = a.ravel(), b.ravel()
    ba, bb = bits(a), bits(b)
    bad = np.flatnonzero(ba != bb)
    # NaNs compare equal regardless of payload
    bad = bad[~(np.isnan(a[bad]) & np.isnan(b[bad]))]
    assert bad.size == 0, (
        f"{what}: {bad.size}/{a.size} differ; first at {bad[0]}: {a[bad[0]]!r} vs {b[bad[0]]!r}")
