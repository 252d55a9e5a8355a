"""The headline configuration's phases vs the oracle, bitwise, with the
production kernels: throughput-mode walks (k_ex0_eval<0,0>, k_lu0_*<0>) with
the no-op tail exit on, the persistent k_moments, the objective integrand.

Controllers: the reference's converged d=2000 solution (golden) linearly
interpolated onto the fine grid -- exactly bench.py's snapshot -- plus the
adversarial stage-1 controllers of tools/tail_exit_ab.py (far-tail spikes,
u1 = y, one 1e200 value whose square overflows).  39-node exhaustion
windows (bench.py / SURVEY.md §8(d) W0).  Every phase runs over the whole
grid on the device; the oracle (reference-order C restatement, pinned to
the reference's goldens) recomputes >= 256 sampled points including both
grid ends.  Reference: solver.py:179-223, kernels.py:406-486, problem.py:110-127.
"""
import numpy as np
import pytest
import torch

from parity_util import assert_bitwise

pytestmark = pytest.mark.gpu

SPAN = (-25.0, 25.0)


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def _snapshot(golden, d, perturb):
    sol = golden("wc_solve_d2000")
    yc = np.linspace(*SPAN, 2000)
    y = np.linspace(*SPAN, d)
    u0 = np.ascontiguousarray(np.interp(y, yc, sol["u0"]))
    u1 = np.ascontiguousarray(np.interp(y, yc, sol["u1"]))
    if perturb == "spike":
        u1[d - 3] = 1e6
        u1[d // 2 + d // 7] = -3e5
        u1[d // 5] = 2e4
    elif perturb == "identity":
        u1 = y.copy()
    elif perturb == "huge":
        u1[d // 2 + d // 9] = 1e200
    return u0, u1


def _points(d, n, seed):
    rng = np.random.default_rng(seed)
    pts = np.unique(np.concatenate([[0, 1, d // 2, d - 2, d - 1], rng.choice(d, n, replace=False)]))
    return pts.astype(np.int64)


def _setup(P, oracle_mod, golden, log2d, perturb):
    d = 1 << log2d
    u0, u1 = _snapshot(golden, d, perturb)
    prob = P.Witsenhausen(k=0.2, sigma=5.0, grids=[(*SPAN, d)] * 2)
    h = prob.grids[0].spacing
    cfg = P.SolverConfig(search_radius=19.5 * h)
    U = P.ControllerSet((P.SampledController(prob.grids[0], u0), P.SampledController(prob.grids[1], u1)))
    p = oracle_mod.OracleWitsenhausen(k=0.2, sigma=5.0, grid0=(*SPAN, d), grid1=(*SPAN, d), f0=prob._f0,
                                      fw0=prob._fw0)
    ocfg = oracle_mod.OracleConfig(search_radius=19.5 * h)
    return d, u0, u1, prob, cfg, U, p, ocfg


@pytest.mark.parametrize("log2d,perturb", [(20, "none"), (18, "none"), (18, "spike"), (18, "identity")])
def test_fine_phases_vs_oracle(P, oracle_mod, golden, log2d, perturb):
    d, u0, u1, prob, cfg, U, p, ocfg = _setup(P, oracle_mod, golden, log2d, perturb)
    pts = _points(d, 300, log2d)
    sh = P.LOCAL
    for m in (0, 1):
        got = P.partial_exhaustion_phase(prob, m, U, cfg, sh)
        want = oracle_mod.partial_exhaustion_phase(p, m, u0, u1, ocfg, points=pts)
        assert_bitwise(got[pts], want, f"EX{m} @2^{log2d} {perturb}")
        got = P.local_update_phase(prob, m, U, cfg, sh)
        want = oracle_mod.local_update_phase(p, m, u0, u1, ocfg, points=pts)
        assert_bitwise(got[pts], want, f"LU{m} @2^{log2d} {perturb}")
    terms = prob.device_objective_terms(U, sh).cpu().numpy()
    assert_bitwise(terms[pts], p.cost_batch(0, u0[pts], pts, u0, u1), f"objective terms @2^{log2d}")
    # J: the device's serial trapezoid == the oracle's over the device integrand
    assert_bitwise(prob.objective(U), oracle_mod.trapezoid_sum(terms, prob.grids[0].spacing), "J")


def test_fine_exhaustion_overflow_error_vs_oracle(P, oracle_mod, golden):
    """u1 holds 1e200: walks reaching it overflow (v*v = inf), the reference raises
    NumericError at the first such grid point.  The device raises the same text;
    the oracle raises it at that point, and sampled points before it are clean."""
    d, u0, u1, prob, cfg, U, p, ocfg = _setup(P, oracle_mod, golden, 18, "huge")
    with pytest.raises(P.NumericError) as ei:
        P.partial_exhaustion_phase(prob, 0, U, cfg)
    msg = str(ei.value)
    bad = int(msg.split("grid point ")[1].split(" ")[0])
    with pytest.raises(oracle_mod.OracleNumericError) as eo:
        oracle_mod.partial_exhaustion_phase(p, 0, u0, u1, ocfg, points=np.array([bad], dtype=np.int64))
    assert str(eo.value) == msg
    before = _points(bad, 64, 3) if bad > 64 else np.arange(bad, dtype=np.int64)
    oracle_mod.partial_exhaustion_phase(p, 0, u0, u1, ocfg, points=before)  # no error below `bad`
    if bad > 0:  # and the oracle agrees the point right before is clean
        oracle_mod.partial_exhaustion_phase(p, 0, u0, u1, ocfg, points=np.array([bad - 1], dtype=np.int64))
