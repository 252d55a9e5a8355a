"""Race shaking (compute-sanitizer is closed on this pool -- gpurun exits 86
for it, profiles/r2_sanitizer_closed.txt): the stress build of the library
(-DUCP_STRESS, paper_1908_04489_b200/_build.py) delays a pseudo-random eighth
of the threads by up to ~2 us around every barrier, named barrier, mbarrier
wait, bulk-copy issue and work-queue fetch, and traps on violated index
invariants (UCP_DCHECK).  tools/sanitize_cases.py drives every kernel family
(latency and throughput walks with the tail exit, both moments kernels, graph-
replayed blocks, the batched engine's work queues, config-5, Monte-Carlo) and
checks the results bitwise against the oracle, so a schedule-dependent race
shows up as a parity failure or a trap.  Each group runs twice (the jitter is
seeded by the clock: different schedules)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def stress_lib():
    from paper_1908_04489_b200 import _build

    return _build.build_stress()


@pytest.mark.parametrize("cases", ["smoke block walk batch c5 mc table tz", "moments"])
@pytest.mark.parametrize("rep", [0, 1])
def test_stress_build_bitwise(stress_lib, cases, rep):
    env = dict(os.environ, UCP_B200_LIB=str(stress_lib), CUDA_LAUNCH_BLOCKING="1")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_cases.py"), *cases.split()], cwd=str(ROOT),
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "UCP_DCHECK failed" not in r.stdout + r.stderr
    for c in cases.split():
        assert f"case {c}: ok" in r.stdout
