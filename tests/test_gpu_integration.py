"""INTEGRATION.md option B: the torch-free `b200` kernel backend a maintainer
would add to the reference (integration/ucpsolve_b200_backend.py) replays the
reference's golden kernel vectors bit for bit."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from parity_util import assert_bitwise

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def kb():
    sys.path.insert(0, str(ROOT / "integration"))
    import ucpsolve_b200_backend as kb

    return kb


@pytest.mark.parametrize("tag", ["k307", "k2", "k64"])
def test_moments_vs_reference_goldens(kb, golden, tag):
    g = golden("kernels")
    a, h, d = float(g[f"{tag}_a"]), float(g[f"{tag}_h"]), int(g[f"{tag}_d"])
    t = kb.gauss_moments_grid(g[f"{tag}_centers"], g[f"{tag}_vals"], a, h, d)
    for k in range(3):
        assert_bitwise(t[k], g[f"{tag}_grid_t{k}"], f"grid T{k}")
    p = kb.gauss_moments_points(g[f"{tag}_queries"], g[f"{tag}_xs"], g[f"{tag}_weights"], a, h, d)
    for k in range(3):
        assert_bitwise(p[k], g[f"{tag}_pts_{k}"], f"points M{k}")


def test_trapezoid_and_argmin_vs_reference_goldens(kb, golden):
    g = golden("kernels")
    assert_bitwise(kb.trapezoid_sum(g["trap_samples"], 0.37), g["trap_value"], "trapezoid")
    got = kb.segmented_argmin(g["argmin_costs"], g["argmin_offsets"])
    assert np.array_equal(got, g["argmin_out"])


def test_backend_needs_no_torch():
    code = ("import sys; sys.path.insert(0, 'integration'); import ucpsolve_b200_backend as kb; "
            "import numpy as np; kb.trapezoid_sum(np.ones(5), 1.0); assert 'torch' not in sys.modules")
    r = subprocess.run([sys.executable, "-c", code], cwd=str(ROOT), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
