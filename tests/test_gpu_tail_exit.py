"""The walk's no-op tail exit (walk_tail_noop in csrc/ucp_kernels.cu) is
result-invariant: every phase output of the bench snapshot and J are bitwise
equal with UCP_TAIL_EXIT=1 (default) and 0 (every node walked, the reference's
loop).  2^17 points: both stage-0 phases run the throughput-mode walk; 2^15:
the exhaustion walks run throughput mode, the local update's latency mode 1;
2^11: latency mode 2 throughout (the switch must be inert there).  A
tail check in the latency-mode loops was tried (shared-memory range-max table
built per CTA): bitwise, but C1 35.1 -> 40.8 ms, so those modes walk every node."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(flag, out, perturb="none", log2d=17):
    env = dict(os.environ, UCP_TAIL_EXIT=flag)
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "tail_exit_ab.py"), "--log2d", str(log2d), "--out",
                        str(out), "--perturb", perturb],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("log2d", [17, 15, 11])
@pytest.mark.parametrize("perturb", ["none", "spike", "identity", "huge"])
def test_tail_exit_bitwise(tmp_path, perturb, log2d):
    """none: the bench snapshot; spike: huge finite u1 values in the far tail (late addends
    that DO change the sums: the exit must not fire before them); identity: u1 = y, so the
    first moment nearly cancels for centres near 0; huge: a 1e200 value (v*v overflows: the bound
    is inf and the walk never ends early; errors must match).  Non-finite controllers never reach
    a walk (SampledController rejects them, as the reference does)."""
    a = _run("0", tmp_path / "full.npz", perturb, log2d)
    b = _run("1", tmp_path / "exit.npz", perturb, log2d)
    assert set(a.files) == set(b.files) == {"local0", "local1", "exh0", "exh1", "J"}
    for k in a.files:
        assert a[k].tobytes() == b[k].tobytes(), k
    if perturb == "none":
        assert b["J"][0] > 0
