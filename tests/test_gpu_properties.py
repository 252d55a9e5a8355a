"""The reference's property tests (pkg/tests/test_problem_core.py,
test_solver.py) run against the device path: marginal-cost consistency,
independence from the stage's own other points, projection, exactly-zero
weights, monotone exhaustion and sweep == brute-force windowed argmin."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1908_04489_b200 as P

    assert torch.cuda.is_available()
    return P


def small_problems(P):
    return {
        "witsenhausen": P.Witsenhausen(grids=[(-25.0, 25.0, 201), (-25.0, 25.0, 201)]),
        "zero_delay": P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)]),
        "inventory": P.Inventory(grids=[(-3.0, 3.0, 241)] * 2),
    }


def perturbed(P, prob, seed=0, scale=0.5):  # reference tests/conftest.py:37-44
    rng = np.random.default_rng(seed)
    return P.ControllerSet(tuple(P.SampledController(g, prob.project(m, g.points + scale * rng.uniform(-1, 1, g.d)))
                                 for m, g in enumerate(prob.grids)))


@pytest.mark.parametrize("name", ["witsenhausen", "zero_delay", "inventory"])
def test_single_point_perturbation_consistency(P, name):
    """dJ == dC * spacing to 1e-6 (test_problem_core.py:9-34)."""
    prob = small_problems(P)[name]
    U = perturbed(P, prob, seed=5)
    rng = np.random.default_rng(11)
    J = prob.objective(U)
    for _ in range(10):
        m = int(rng.integers(0, prob.M))
        g = prob.grids[m]
        i = int(rng.integers(0, g.d))
        y, u_old = float(g.points[i]), float(U.values(m)[i])
        vals = U.values(m).copy()
        vals[i] = u_old + 0.05
        J2 = prob.objective(U.replace(m, U[m].with_values(vals)))
        dC = prob.marginal_cost(m, u_old + 0.05, y, U) - prob.marginal_cost(m, u_old, y, U)
        assert abs((J2 - J) - dC * g.spacing) / (1.0 + abs(J)) <= 1e-6


@pytest.mark.parametrize("name", ["witsenhausen", "zero_delay", "inventory"])
def test_marginal_cost_ignores_own_other_points(P, name):
    prob = small_problems(P)[name]
    U = perturbed(P, prob, seed=6)
    rng = np.random.default_rng(7)
    for m in range(prob.M):
        g = prob.grids[m]
        i = int(rng.integers(1, g.d - 1))
        y, u = float(g.points[i]), float(U.values(m)[i]) + 0.3
        before = prob.marginal_cost(m, u, y, U)
        vals = U.values(m).copy()
        vals[(i + 5) % g.d] += 1.7
        assert prob.marginal_cost(m, u, y, U.replace(m, U[m].with_values(vals))) == before


def test_witsenhausen_tail_weight_exactly_zero(P):
    wc = small_problems(P)["witsenhausen"]
    U = wc.zero_controllers()
    U = U.replace(0, U[0].with_values(-wc.grids[0].points))
    J = wc.objective(U)
    vals = U.values(1).copy()
    vals[-1] = 9.0
    assert wc.objective(U.replace(1, U[1].with_values(vals))) == J


def test_inventory_zero_weight_points(P):
    inv = small_problems(P)["inventory"]
    U = inv.identity_controllers()
    U = P.ControllerSet(tuple(P.SampledController(g, inv.project(m, U.values(m))) for m, g in enumerate(inv.grids)))
    J = inv.objective(U)
    g = inv.grids[0]
    i = int(np.argmin(np.abs(g.points - 2.5)))
    vals = U.values(0).copy()
    vals[i] += 3.0
    assert inv.objective(U.replace(0, U[0].with_values(vals))) == J


@pytest.mark.parametrize("name", ["witsenhausen", "zero_delay", "inventory"])
def test_exhaustion_is_monotone_and_matches_bruteforce(P, name):
    """Exhaustion never raises J (test_solver.py:191-200) and equals the
    per-point windowed argmin done with scalar evaluations (oracle.py:66-95)."""
    prob = small_problems(P)[name]
    U = perturbed(P, prob, seed=3, scale=1.0)
    cfg = P.SolverConfig()
    J0 = prob.objective(U)
    V = P.run_block(prob, U, cfg, 1, "exhaustion")
    assert prob.objective(V) <= J0
    m = 0
    g = prob.grids[m]
    new = P.partial_exhaustion_phase(prob, m, U, cfg)
    r = cfg.radius_for(g)
    for i in np.random.default_rng(1).choice(g.d, 12, replace=False):
        y = float(g.points[i])
        best_u, best_c = math.nan, math.inf
        for j in P.window_indices(g, y, r):
            u = float(U.values(m)[j])
            if u == best_u:
                continue
            c = prob.marginal_cost(m, u, y, U)
            if c < best_c:
                best_c, best_u = c, u
        assert prob.project(m, np.array([best_u]))[0] == new[i]


def test_local_update_closed_form_quadratic_stage(P):
    """Stage-1 cost is exactly quadratic in u, so one Newton step lands on B/A
    (test_solver.py:135-145 analogue), up to the monotone guard."""
    wc = small_problems(P)["witsenhausen"]
    U = perturbed(P, wc, seed=2)
    new1 = P.local_update_phase(wc, 1, U, P.SolverConfig())
    # minimiser of A u^2 - 2 B u + C from three costs per point
    y = wc.grids[1].points
    c_at = lambda u: wc.marginal_cost_batch(1, np.full(y.size, u), y, U)  # noqa: E731
    c0, c1, c2 = c_at(0.0), c_at(1.0), c_at(-1.0)
    A = (c1 + c2 - 2 * c0) / 2.0
    B = (c2 - c1) / 4.0
    np.testing.assert_allclose(new1, B / A, rtol=5e-3, atol=5e-3)


def test_solve_determinism_and_warm_start(P):
    wc = P.Witsenhausen(grids=[(-25.0, 25.0, 151)] * 2)
    a = P.solve(wc, P.SolverConfig(max_rounds=3))
    b = P.solve(wc, P.SolverConfig(max_rounds=3))
    assert a.final_objective == b.final_objective
    assert np.array_equal(np.asarray(a.controllers.values(0)), np.asarray(b.controllers.values(0)))
    c = P.solve(wc, P.SolverConfig(max_rounds=2), initial=a.controllers)
    assert c.rounds[0].objective <= a.final_objective
