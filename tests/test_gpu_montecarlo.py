"""Monte-Carlo objective on the device.

* the reference's estimator (host PCG64 draws, device costs) is bitwise the
  reference's recorded costs and (estimate, stderr);
* the device generator (Philox4x32-10) matches the oracle's restatement --
  uniforms bitwise, Box-Muller normals to a few ulp -- and the device
  estimate equals the oracle's fixed-order reduction of the device costs
  bit for bit;
* statistical agreement with the quadrature objective: the reference's own
  tests (test_oracle.py:73-99) and acceptance criterion 8.
"""
import math

import numpy as np
import pytest
import torch

from mc_cases import CASES, SEEDS, ReplayRng, controllers, device_problem, oracle_problem
from parity_util import assert_bitwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


def _U(P, prob, g, tag):
    return P.ControllerSet(tuple(P.SampledController(gr, u)
                                 for gr, u in zip(prob.grids, controllers(g, tag, prob.M))))


@pytest.mark.parametrize("tag", CASES)
def test_simulate_cost_bitwise(P, golden, tag):
    g = golden("mc")
    prob = device_problem(P, tag)
    U = _U(P, prob, g, tag)
    costs = prob.simulate_cost(U, ReplayRng(g[f"{tag}_draws"]), 2000)
    assert_bitwise(costs, g[f"{tag}_costs"], f"{tag} device costs")


@pytest.mark.parametrize("tag", CASES)
def test_reference_estimator_bitwise(P, golden, tag):
    g = golden("mc")
    prob = device_problem(P, tag)
    U = _U(P, prob, g, tag)
    for n, seed in ((2000, SEEDS[tag]), (100_000, 7)):
        got = P.monte_carlo_objective(prob, U, P.OracleConfig(mc_samples=n, seed=seed))
        assert_bitwise(np.array(got), g[f"{tag}_mc_{n}_{seed}"], f"{tag} mc n={n}")


@pytest.mark.parametrize("tag", CASES)
def test_philox_draws_match_restatement(P, golden, oracle_mod, tag):
    from paper_1908_04489_b200.montecarlo import philox_draws

    g = golden("mc")
    prob = device_problem(P, tag)
    U = _U(P, prob, g, tag)
    p = oracle_problem(oracle_mod, tag)
    for seed, begin, end in ((0, 0, 5000), (2**40 + 17, 2**33 - 100, 2**33 + 900)):
        dev = philox_draws(prob, U, seed, begin, end)
        ref = oracle_mod.philox_draws(p, seed, begin, end)
        assert dev.shape == ref.shape
        normal_streams = {"wc": (0, 1), "zd": (0,)}.get(tag, ())
        for s in range(dev.shape[0]):
            if s in normal_streams:
                np.testing.assert_allclose(dev[s], ref[s], rtol=0, atol=64 * np.finfo(float).eps * 40)
            else:
                assert_bitwise(dev[s], ref[s], f"{tag} uniform stream {s}")


@pytest.mark.parametrize("tag", CASES)
@pytest.mark.parametrize("n", [1, 2, 4095, 4097, 123_457])
def test_device_estimator_fixed_order(P, golden, oracle_mod, tag, n):
    """estimate/stderr == the oracle's restatement of the fixed-order
    reduction over the device's own per-sample costs (bitwise)."""
    from paper_1908_04489_b200.montecarlo import philox_draws

    g = golden("mc")
    prob = device_problem(P, tag)
    U = _U(P, prob, g, tag)
    seed = 2024 + n
    draws = philox_draws(prob, U, seed, 0, n)
    costs = prob.simulate_cost(U, ReplayRng(draws), n)  # buffer draws -> same kernel cost function
    p = oracle_problem(oracle_mod, tag)
    assert_bitwise(costs, oracle_mod.simulate_cost(p, controllers(g, tag, p.M), draws), "costs vs oracle")
    est, se = P.device_monte_carlo_objective(prob, U, n, seed=seed)
    if n == 1:
        assert est == costs[0] and math.isnan(se)
        return
    want = oracle_mod.mc_estimate(costs)
    assert_bitwise(np.array([est, se]), np.array(want), "device estimate vs fixed-order restatement")


def test_device_estimator_reproducible_and_seeded(P):
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    U = prob.identity_controllers()
    a = P.device_monte_carlo_objective(prob, U, 1_000_003, seed=77)
    b = P.device_monte_carlo_objective(prob, U, 1_000_003, seed=77)
    c = P.device_monte_carlo_objective(prob, U, 1_000_003, seed=78)
    assert a == b and a != c


def test_known_answers_zero_controllers(P):
    """test_oracle.py:73-82: zero controllers give J = sigma^2 = 25 and 1."""
    wc = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    zd = P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)])
    for prob, J, seed in ((wc, 25.0, 5), (zd, 1.0, 6)):
        est, se = P.monte_carlo_objective(prob, prob.zero_controllers(), P.OracleConfig(mc_samples=10**6, seed=seed))
        assert abs(est - J) <= 4 * se
        est, se = P.device_monte_carlo_objective(prob, prob.zero_controllers(), 10**8, seed=seed)
        assert abs(est - J) <= 4 * se


@pytest.mark.parametrize("tag", ["wc", "zd", "inv"])
def test_agrees_with_quadrature(P, tag):
    """test_oracle.py:92-99: perturbed controllers, |J - est| <= 5 se."""
    prob = device_problem(P, tag)
    for seed in (41, 42, 43):
        rng = np.random.default_rng(seed)
        U = P.ControllerSet(tuple(P.SampledController(g, prob.project(m, g.points + 0.3 * rng.uniform(-1, 1, g.d)))
                                  for m, g in enumerate(prob.grids)))
        J = prob.objective(U)
        est, se = P.monte_carlo_objective(prob, U, P.OracleConfig(mc_samples=300_000, seed=seed))
        assert abs(J - est) <= 5 * se
        est, se = P.device_monte_carlo_objective(prob, U, 300_000, seed=seed)
        assert abs(J - est) <= 5 * se


def test_criterion_8_quadrature_vs_monte_carlo(P):
    """test_acceptance.py:291-302 on the default problems, both estimators."""
    for prob in (P.Witsenhausen(), P.ZeroDelay()):
        for U in (prob.zero_controllers(), prob.identity_controllers()):
            J = prob.objective(U)
            est, se = P.monte_carlo_objective(prob, U, P.OracleConfig(mc_samples=10**6, seed=8))
            assert abs(J - est) <= 5 * se
            est, se = P.device_monte_carlo_objective(prob, U, 10**6, seed=8)
            assert abs(J - est) <= 5 * se


def test_bad_arguments(P):
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, 201)] * 2)
    with pytest.raises(ValueError):
        P.device_monte_carlo_objective(prob, prob.zero_controllers(), 0)
    other = P.Witsenhausen(grids=[(-25.0, 25.0, 101)] * 2)
    with pytest.raises(ValueError):
        P.device_monte_carlo_objective(prob, other.zero_controllers(), 10)
